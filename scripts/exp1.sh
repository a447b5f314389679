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
one fused WS_EXP=0
one fused_fence0 WS_EXP=2
one fused_noborder WS_EXP=1
one fused_noborder_fence0 WS_EXP=3
one nofuse WS_NOFUSE=1
CMD="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu"
WS_NOFUSE=1 $CMD > gpurun_out/plain_nf.log 2>&1 && WS_NOFUSE=1 ncu --set full --clock-control none --import-source on -k regex:k_speeds -s 4 -c 1 -o gpurun_out/prof_speeds2 $CMD > gpurun_out/ncu_sp2.log 2>&1
echo ncu_rc=$?
$CMD > gpurun_out/plain_f.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_update -s 4 -c 1 -o gpurun_out/prof_update_fused $CMD > gpurun_out/ncu_uf.log 2>&1
echo ncu2_rc=$?
