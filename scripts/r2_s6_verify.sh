# session-6 re-entry check of the per-solver line-kernel policy: the GPU suite, then one bench line per config
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s6_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -n 2 gpurun_out/s6_pytest_gpu.log
for c in c5 c4 c3 c2 c1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-ref-code > gpurun_out/s6_$c.json 2> gpurun_out/s6_$c.err
  python - gpurun_out/s6_$c.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(r['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
done
