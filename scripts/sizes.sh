# per-cell cost vs grid size (small-grid overheads): c2 and c5 physics
for cfg in "c2 1024" "c2 2048" "c2 4096" "c5 1024" "c5 4096"; do
set -- $cfg
timeout 900 python bench.py --config $1 --size $2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/sz.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/sz.log').read().strip().split('\n')[-1])
r=d['roofline']; n=d['config']['nx']*d['config']['ny']
print('$1 $2', 'Gcell/s %.2f'%(d['value']/1e9), 'upd ps/cell %.1f'%(r['kernel_ms']*1e9/n), 'spd ps/cell %.1f'%(r['speeds_kernel_ms']*1e9/n))
" || tail -3 gpurun_out/sz.log
done
