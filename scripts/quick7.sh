# pytest -m gpu, then C2 bench twice (A/B noise check)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? ; tail -2 gpurun_out/pytest_gpu.log
for rep in 1 2; do
timeout 600 python bench.py --config c2 --steps 30 --warmup 5 --no-e2e --no-cpu ${BENCH_ENV:-} > gpurun_out/b7_$rep.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/b7_$rep.log').read().strip().split('\n')[-1])
r=d['roofline']
print('c2', 'Gcell/s %.3f'%(d['value']/1e9), 'update_ms %.4f'%r['kernel_ms'], 'speeds_ms %.4f'%r['speeds_kernel_ms'], 'sim %.3f'%(d['simulation']['cell_updates_per_s']/1e9))
" || tail -3 gpurun_out/b7_$rep.log
done
WS_SPEEDS=smem timeout 600 python bench.py --config c2 --steps 30 --warmup 5 --no-e2e --no-cpu > gpurun_out/b7_smem.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/b7_smem.log').read().strip().split('\n')[-1])
r=d['roofline']
print('c2 smem-prepass', 'Gcell/s %.3f'%(d['value']/1e9), 'update_ms %.4f'%r['kernel_ms'], 'speeds_ms %.4f'%r['speeds_kernel_ms'])
"
