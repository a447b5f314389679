timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? ; tail -3 gpurun_out/pytest_gpu.log
for c in c2 c3 c4; do
timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/b5_$c.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/b5_$c.log').read().strip().split('\n')[-1])
r=d['roofline']
print('$c', 'Gcell/s %.3f'%(d['value']/1e9), 'update_ms %.4f'%r['kernel_ms'], 'speeds_ms %.4f'%r['speeds_kernel_ms'], 'sim %.3f'%(d['simulation']['cell_updates_per_s']/1e9), 'frac %.3f'%r['frac'])
" || tail -3 gpurun_out/b5_$c.log
done
