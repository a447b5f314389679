for c in c2 c3; do timeout 600 python bench.py --config $c --force-sharded --strong --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/st_$c.json 2>&1; tail -c 400 gpurun_out/st_$c.json; echo; done
timeout 900 python bench.py --config c5 --force-sharded --strong --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/st_c5.json 2>&1; tail -c 400 gpurun_out/st_c5.json; echo
timeout 600 python -m pytest tests/test_gpu_nccl1.py -q > gpurun_out/pytest_nccl.log 2>&1; echo rc=$?; tail -n 2 gpurun_out/pytest_nccl.log
