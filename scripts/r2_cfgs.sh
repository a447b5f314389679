# round 2: graph-replay suites again, bench lines of every config (no CPU / e2e
# legs), ncu full capture of the C4 and C3 update kernels
timeout 900 python -m pytest tests/test_gpu_multishard.py tests/test_gpu_nccl1.py -q -x > gpurun_out/r2c_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2c_pytest.log
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2c_$c.json 2> gpurun_out/r2c_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --config c3 --precision f32 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2c_c3_f32.json 2> gpurun_out/r2c_c3_f32.err
timeout 900 python bench.py --config c5 --precision f32 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2c_c5_f32.json 2> gpurun_out/r2c_c5_f32.err; echo "c5f32 rc=$?"
for c in c4 c3; do
CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu"
ncu --set full --clock-control none --import-source on -k regex:"k_update_w" -s 4 -c 1 -o gpurun_out/r2c_prof_$c $CMD > gpurun_out/r2c_ncu_$c.log 2>&1
echo ncu_$c rc=$?
ncu -i gpurun_out/r2c_prof_$c.ncu-rep --page raw --csv > gpurun_out/r2c_raw_$c.csv 2>/dev/null
ncu -i gpurun_out/r2c_prof_$c.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2c_src_$c.csv 2>/dev/null
done
for f in gpurun_out/r2c_c*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value']/1e9, d['ms_per_step'], d['roofline'].get('kernel_ms'), d.get('simulation',{}).get('cell_updates_per_s',0)/1e9)"; done
