# A/B of the L2 band prefetch (WS_L2PF=1; vpf: 444 CTAs ahead, vpf9: 900) vs default, then parity on vpf
ab() {
  if [ -n "$2" ]; then export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/$2/libwavestep.so; else unset WAVESTEP_LIB; fi
  timeout 600 python bench.py --config $3 --precision $4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-ref-code > gpurun_out/ab7_$1.json 2> gpurun_out/ab7_$1.err
  python - gpurun_out/ab7_$1.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(r['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
}
for c in c4 c5 c3 c2; do for v in "" ${VARIANTS:-vpf vpf9}; do ab ${c}_f64_${v:-def} "$v" $c f64; done; done
for c in c4 c5; do for v in "" ${VARIANTS:-vpf vpf9}; do ab ${c}_f32_${v:-def} "$v" $c f32; done; done
export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/${PARITY_VARIANT:-vpf}/libwavestep.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_recipes.py tests/test_gpu_multishard.py -q -x > gpurun_out/ab7_parity.log 2>&1; echo parity_rc=$?; tail -n 3 gpurun_out/ab7_parity.log
