# round-end style evidence run: tests, smoke, bench (both arms), ncu launch list + full capture
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/o_pytest_gpu.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/o_smoke.log 2>&1; echo smoke_rc=$?
./tools/fp64_peak > gpurun_out/o_fp64_peak.json 2>&1
python bench.py > gpurun_out/o_bench.json 2> gpurun_out/o_bench.err; echo bench_rc=$?
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/o_bench_ref.json 2> gpurun_out/o_bench_ref.err; echo ref_rc=$?
# launch list of the exact default bench command (it exited 0 just above)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/o_launches.csv python bench.py > gpurun_out/o_ncu_launch.log 2>&1
echo launch_rc=$?
CMD="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/o_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_update_w|k_speeds|k_tiles" -s 12 -c 3 -o gpurun_out/o_prof $CMD > gpurun_out/o_ncu_full.log 2>&1
echo full_rc=$?
ncu -i gpurun_out/o_prof.ncu-rep --page raw --csv > gpurun_out/o_raw.csv 2>/dev/null
ncu -i gpurun_out/o_prof.ncu-rep --page details --csv > gpurun_out/o_details.csv 2>/dev/null
ncu -i gpurun_out/o_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/o_src.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
tail -3 gpurun_out/o_pytest_gpu.log; cat gpurun_out/o_smoke.log; cat gpurun_out/o_bench.json; cat gpurun_out/o_bench_ref.json
