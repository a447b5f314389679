timeout 600 python -m pytest tests/test_gpu_multishard.py tests/test_gpu_nccl1.py -q > gpurun_out/pytest_shard.log 2>&1; echo rc=$?; tail -n 15 gpurun_out/pytest_shard.log
for f in "" "--device-reduce" "--device-reduce --device-halo"; do timeout 300 python bench.py --force-sharded $f --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/shb.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/shb.json').read().strip().splitlines()[-1]); print('$f', d['value']/1e9, d['ms_per_step'])"; done
