timeout 300 python -m pytest tests/test_gpu_cfl_filter.py -x -q > gpurun_out/pytest_filter.log 2>&1; echo filter_rc=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -n 3 gpurun_out/pytest_filter.log; tail -n 5 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
