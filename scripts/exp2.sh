for e in 0 1 2 4 7; do WS_EXP=$e timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/e2_$e.json 2>&1; done
WS_SPEEDS=exact timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/e2_x.json 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/e2_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["value"]/1e9,3), d["ms_per_step"], d["roofline"].get("kernel_ms"), d["roofline"].get("speeds_kernel_ms"))
    except Exception as e: print(f, "ERR", open(f).read()[-500:])
PY
