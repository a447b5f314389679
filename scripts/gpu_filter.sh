timeout 900 python -m pytest tests/test_gpu_cfl_filter.py -q > gpurun_out/pytest_filter.log 2>&1; echo rc=$?; tail -n 15 gpurun_out/pytest_filter.log
