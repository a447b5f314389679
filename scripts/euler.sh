timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -n 3 gpurun_out/pytest_gpu.log
for v in tile exact; do WS_SPEEDS=$v timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/eu_c3_$v.json 2>&1; done
WS_SPEEDS=tile timeout 600 python bench.py --config c3 --precision f32 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/eu_c3f32_tile.json 2>&1
WS_SPEEDS=exact timeout 600 python bench.py --config c3 --precision f32 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/eu_c3f32_exact.json 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/eu_c2.json 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/eu_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["value"]/1e9,3), d["roofline"].get("kernel_ms"), d["roofline"].get("speeds_kernel_ms"))
    except Exception as e: print(f, "ERR", open(f).read()[-300:])
PY
