timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -n 3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/cph_c2.json 2>&1
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/cph_c3.json 2>&1
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/cph_c5.json 2>&1
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/cph_c4.json 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/cph_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["value"]/1e9,3), d["ms_per_step"], d["roofline"].get("kernel_ms"), d["roofline"].get("speeds_kernel_ms"))
PY
