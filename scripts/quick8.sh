# pytest -m gpu, then the bench per environment variant (VARIANTS, CFG)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? ; tail -2 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-"WS_PDL=1" "WS_SPEEDS=smem" "WS_PDL=0"}; do
env $v timeout 600 python bench.py --config ${CFG:-c2} --steps 30 --warmup 5 --no-e2e --no-cpu > gpurun_out/b8.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/b8.log').read().strip().split('\n')[-1])
r=d['roofline']
print('$v', 'Gcell/s %.3f'%(d['value']/1e9), 'update_ms %.4f'%r['kernel_ms'], 'speeds_ms %.4f'%r['speeds_kernel_ms'], 'sim %.3f'%(d['simulation']['cell_updates_per_s']/1e9))
" || tail -3 gpurun_out/b8.log
done
