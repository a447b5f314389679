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
one tile WS_KERNEL=tile
CMD="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_l.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_update_w|k_speeds" -s 8 -c 2 -o gpurun_out/prof_line $CMD > gpurun_out/ncu_line.log 2>&1
echo ncu_rc=$?
for k in k_update_w k_speeds; do
  ncu -i gpurun_out/prof_line.ncu-rep -k regex:$k --page raw --csv > gpurun_out/raw_$k.csv 2>/dev/null
  ncu -i gpurun_out/prof_line.ncu-rep -k regex:$k --page source --csv --print-source cuda,sass > gpurun_out/src_$k.csv 2>/dev/null
done
ls -la gpurun_out/
rm -f gpurun_out/*.ncu-rep
