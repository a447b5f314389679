timeout 300 python -m pytest tests/test_gpu_multishard.py tests/test_gpu_cfl_filter.py tests/test_gpu_nccl1.py -x -q > gpurun_out/pytest_shard.log 2>&1; echo shard_rc=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python bench.py --force-sharded --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_sharded.json 2>&1; echo sh_rc=$?
tail -n 3 gpurun_out/pytest_shard.log; tail -n 5 gpurun_out/pytest_gpu.log; tail -c 600 gpurun_out/bench_sharded.json
