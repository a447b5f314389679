# A/B: 10-warp line kernel at 3 CTAs/SM (<= 64 regs, 72 KB smem; default build)
# vs 2 CTAs/SM (WS_LB3=0 build in _lib/lb2), both with the dimension-by-dimension update
for cfg in c5 c4 c2 c3; do
  for v in lb3 lb2; do
    if [ $v = lb2 ]; then export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/lb2/libwavestep.so; else unset WAVESTEP_LIB; fi
    python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu --no-ref-code > gpurun_out/lb_${cfg}_$v.json 2> gpurun_out/lb_${cfg}_$v.err
    python - gpurun_out/lb_${cfg}_$v.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(d['roofline']['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
  done
done
unset WAVESTEP_LIB
python bench.py --config c5 --precision f32 --steps 20 --warmup 5 --no-e2e --no-cpu --no-ref-code > gpurun_out/lb_c5f32.json 2>&1; tail -c 300 gpurun_out/lb_c5f32.json
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/lb_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/lb_pytest.log
