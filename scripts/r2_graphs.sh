# round 2: graph-replayed sharded steps (StepGraph over NCCL, ws_run for
# device-collective shards), multishard + NCCL world-1 suites, sharded C5 lines
set -x
timeout 900 python -m pytest tests/test_gpu_multishard.py tests/test_gpu_nccl1.py -q -x > gpurun_out/r2g_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r2g_pytest.log
for extra in "" "--eager" "--device-reduce" "--device-halo"; do
  timeout 600 python bench.py --force-sharded --steps 10 --warmup 3 --no-e2e --no-cpu $extra > gpurun_out/r2g_sharded$(echo $extra | tr -d ' -').json 2> gpurun_out/r2g_sharded_err$(echo $extra | tr -d ' -').log; echo "sharded $extra rc=$?"
  cut -c1-400 gpurun_out/r2g_sharded$(echo $extra | tr -d ' -').json
  tail -3 gpurun_out/r2g_sharded_err$(echo $extra | tr -d ' -').log
done
