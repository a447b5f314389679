timeout 600 python -m pytest tests -m gpu -q -k "fp32 or f32 or euler" > gpurun_out/pytest_f32.log 2>&1; echo rc=$?; tail -n 2 gpurun_out/pytest_f32.log
for v in tile exact; do WS_SPEEDS=$v timeout 600 python bench.py --config c3 --precision f32 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/f32_c3_$v.json 2>&1; done
timeout 600 python bench.py --config c5 --precision f32 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/f32_c5.json 2>&1
timeout 600 python bench.py --config c2 --precision f32 --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/f32_c2.json 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/f32_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["value"]/1e9,3), d["roofline"].get("kernel_ms"), d["roofline"].get("speeds_kernel_ms"))
    except Exception as e: print(f, "ERR", open(f).read()[-400:])
PY
