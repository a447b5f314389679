timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? ; tail -5 gpurun_out/pytest_gpu.log
one() {  # label env...
  label=$1; shift
  env "$@" timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu > gpurun_out/exp_$label.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/exp_$label.log').read().strip().split('\n')[-1])
r=d['roofline']
print('$label', 'Gcell/s %.3f'%(d['value']/1e9), 'update_ms %.4f'%r['kernel_ms'], 'speeds_ms %.4f'%r['speeds_kernel_ms'], 'sim %.3f'%(d['simulation']['cell_updates_per_s']/1e9))
" || tail -3 gpurun_out/exp_$label.log
}
one line WS_EXP=0
for c in c1 c3 c4; do label=$c; env WS_EXP=0 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/exp_$c.log 2>&1; tail -c 600 gpurun_out/exp_$c.log; echo ; done
