timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? ; tail -5 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-0 2}; do
  WS_TILE=$v timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu > gpurun_out/tile_$v.log 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/tile_$v.log').read().strip().split('\n')[-1])
r=d['roofline']
print('variant $v', 'Gcell/s %.3f'%(d['value']/1e9), 'update_ms %.4f'%r['kernel_ms'], 'speeds_ms %.4f'%r['speeds_kernel_ms'], 'sim Gcell/s %.3f'%(d['simulation']['cell_updates_per_s']/1e9), d['clocks'], 'launches', d['gpu_launches'])
" || tail -3 gpurun_out/tile_$v.log
done
