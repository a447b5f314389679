# f32fast with -ftz=true: tests + lines
timeout 900 python -m pytest tests/test_gpu_fp32fast.py tests/test_gpu_checked.py -q -x -s > gpurun_out/ftz_pytest.log 2>&1; echo pytest_rc=$?
grep -E "rel|passed|failed|Error" gpurun_out/ftz_pytest.log | head -20
for c in c5 c3 c4 c2; do
  timeout 600 python bench.py --config $c --precision f32fast --steps 10 --warmup 3 --no-cpu --no-e2e --no-ref-code > gpurun_out/ftz_$c.json 2> gpurun_out/ftz_$c.err
  python - gpurun_out/ftz_$c.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(r['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
done
