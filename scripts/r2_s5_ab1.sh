# A/B of the session-5 line-kernel knobs: WS_LIMSEL, WS_ROWSTAGE, WS_ROWSTORE (each alone, all three) vs default
ab() {
  if [ -n "$2" ]; then export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/$2/libwavestep.so; else unset WAVESTEP_LIB; fi
  timeout 600 python bench.py --config $3 --precision $4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-ref-code > gpurun_out/ab5_$1.json 2> gpurun_out/ab5_$1.err
  python - gpurun_out/ab5_$1.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(r['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
}
for c in c5 c4 c2 c3; do for v in "" ${VARIANTS:-vlim vstage vstore vall}; do ab ${c}_f64_${v:-def} "$v" $c f64; done; done
for v in "" ${VARIANTS:-vlim vstage vstore vall}; do ab c5_f32_${v:-def} "$v" c5 f32; done
export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/${PARITY_VARIANT:-vall}/libwavestep.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_recipes.py tests/test_gpu_run_small.py -q -x > gpurun_out/ab5_parity.log 2>&1; echo parity_rc=$?; tail -3 gpurun_out/ab5_parity.log
