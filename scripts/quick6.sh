timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? ; tail -3 gpurun_out/pytest_gpu.log
for f in 1 0; do
WS_FUSE=$f timeout 600 python bench.py --config c2 --steps 30 --warmup 3 --no-e2e --no-cpu > gpurun_out/b6_$f.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/b6_$f.log').read().strip().split('\n')[-1])
r=d['roofline']
print('fuse=$f', 'Gcell/s %.3f'%(d['value']/1e9), 'ms/step %.4f'%d['ms_per_step'], 'update_ms %.4f'%r['kernel_ms'], 'speeds_ms %.4f'%r['speeds_kernel_ms'], 'sim %.3f'%(d['simulation']['cell_updates_per_s']/1e9), 'launches', d['gpu_launches'])
" || tail -3 gpurun_out/b6_$f.log
done
