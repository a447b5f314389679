# round 2, first GPU pass: full GPU suite (incl. the BASELINE recipe parity
# tests), smoke, C5 bench (both arms, driver flags), ncu launch list of the
# default command and one full capture of the C5 step kernels
set -x
nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/r2_pytest_gpu.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke_rc=$?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo ref_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5.csv python bench.py --steps 20 --warmup 5 > gpurun_out/r2_ncu_launch.log 2>&1
echo launch_rc=$?
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/r2_plain.log 2>&1; echo plain_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_update_w|k_speeds" -s 6 -c 2 -o gpurun_out/r2_prof_c5 $CMD > gpurun_out/r2_ncu_full.log 2>&1
echo full_rc=$?
ncu -i gpurun_out/r2_prof_c5.ncu-rep --page raw --csv > gpurun_out/r2_raw_c5.csv 2>/dev/null
ncu -i gpurun_out/r2_prof_c5.ncu-rep --page details --csv > gpurun_out/r2_details_c5.csv 2>/dev/null
ncu -i gpurun_out/r2_prof_c5.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2_src_c5.csv 2>/dev/null
tail -40 gpurun_out/r2_pytest_gpu.log; cat gpurun_out/r2_smoke.log; cat gpurun_out/r2_bench.json; cat gpurun_out/r2_bench_ref.json
grep -E "Elapsed|Maximum resident" gpurun_out/r2_bench.err gpurun_out/r2_bench_ref.err
