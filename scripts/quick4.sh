./tools/check_fastmath $((1<<28)); echo check_rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? ; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu > gpurun_out/b4.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/b4.log').read().strip().split('\n')[-1])
r=d['roofline']
print('Gcell/s %.3f'%(d['value']/1e9), 'update_ms %.4f'%r['kernel_ms'], 'speeds_ms %.4f'%r['speeds_kernel_ms'], 'sim %.3f'%(d['simulation']['cell_updates_per_s']/1e9))
"
