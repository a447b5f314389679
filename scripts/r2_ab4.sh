# A/B: 3-component fp64 line kernel at 2 x 15-warp CTAs per SM (_lib/w15) vs 3 x 10 (default); checked cases
ab() {
  if [ -n "$2" ]; then export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/$2/libwavestep.so; else unset WAVESTEP_LIB; fi
  timeout 600 python bench.py --config $3 --precision $4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-ref-code > gpurun_out/ab4_$1.json 2> gpurun_out/ab4_$1.err
  python - gpurun_out/ab4_$1.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(r['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
}
for c in c5 c4 c2; do ab ${c}_def "" $c f64; ab ${c}_w15 w15 $c f64; done
unset WAVESTEP_LIB
timeout 900 python -m pytest tests/test_gpu_checked.py -q -x > gpurun_out/ab4_checked.log 2>&1; echo checked_rc=$?; tail -3 gpurun_out/ab4_checked.log
WAVESTEP_LIB=paper_1308_1464_b200/_lib/checked/libwavestep.so python tests/checked_cases.py 2>&1 | grep -E "f32fast|256x256|100x90|false" | head
