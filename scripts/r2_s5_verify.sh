# session-5 re-entry check: the GPU suite, the default bench line and the reference arm
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5_smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s5_pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 900 python bench.py > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5_bench_ref.json 2> gpurun_out/s5_bench_ref.err; echo ref_rc=$?
tail -n 3 gpurun_out/s5_smoke.log gpurun_out/s5_pytest_gpu.log; tail -c 1500 gpurun_out/s5_bench.json; tail -c 600 gpurun_out/s5_bench_ref.json
