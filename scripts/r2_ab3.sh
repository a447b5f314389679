# A/B: line kernel staging with cp.async straight into shared memory (_lib/sasync) vs registers (default)
ab() {
  if [ -n "$2" ]; then export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/$2/libwavestep.so; else unset WAVESTEP_LIB; fi
  timeout 600 python bench.py --config $3 --precision $4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-ref-code > gpurun_out/ab3_$1.json 2> gpurun_out/ab3_$1.err
  python - gpurun_out/ab3_$1.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(r['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
}
for c in c4 c5 c2 c3; do ab ${c}_def "" $c f64; ab ${c}_sa sasync $c f64; done
ab c5f_def "" c5 f32fast; ab c5f_sa sasync c5 f32fast
export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/sasync/libwavestep.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_recipes.py -q -x > gpurun_out/ab3_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/ab3_pytest.log
