timeout 900 python -m pytest tests/test_gpu_multishard.py tests/test_gpu_nccl1.py tests/test_gpu_checked.py -q -x > gpurun_out/sh_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/sh_pytest.log
python bench.py --force-sharded --steps 20 --warmup 5 --no-ref-code > gpurun_out/sh_c5.json 2> gpurun_out/sh_c5.err; echo c5_rc=$?; tail -c 1500 gpurun_out/sh_c5.json; tail -5 gpurun_out/sh_c5.err
python bench.py --force-sharded --config c2 --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/sh_c2.json 2> gpurun_out/sh_c2.err; echo c2_rc=$?; tail -c 600 gpurun_out/sh_c2.json
