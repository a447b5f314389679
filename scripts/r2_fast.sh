# fp32 throughput mode: tests, C5 / C3 lines in both fp32 modes
timeout 900 python -m pytest tests/test_gpu_fp32fast.py -q -x -s > gpurun_out/fast_pytest.log 2>&1; echo pytest_rc=$?
grep -E "rel|passed|failed|Error" gpurun_out/fast_pytest.log | head -30
for p in f32 f32fast; do
  for c in c5 c3; do
    timeout 600 python bench.py --config $c --precision $p --steps 10 --warmup 3 --no-cpu --no-e2e --no-ref-code > gpurun_out/fast_${c}_$p.json 2> gpurun_out/fast_${c}_$p.err
    python - gpurun_out/fast_${c}_$p.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(r['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
  done
done
