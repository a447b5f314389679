# fp32 line kernel at 4 CTAs/SM (default now) vs 3 (_lib/base): exact and fast fp32; full GPU suite
ab() {
  if [ -n "$2" ]; then export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/$2/libwavestep.so; else unset WAVESTEP_LIB; fi
  timeout 600 python bench.py --config $3 --precision $4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-ref-code > gpurun_out/ab2_$1.json 2> gpurun_out/ab2_$1.err
  python - gpurun_out/ab2_$1.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(r['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
}
ab c5f32_base base c5 f32; ab c5f32_new "" c5 f32
ab c5fast_base base c5 f32fast; ab c5fast_new "" c5 f32fast
ab c4f32_base base c4 f32; ab c4f32_new "" c4 f32
unset WAVESTEP_LIB
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/ab2_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/ab2_pytest.log
