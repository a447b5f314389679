timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -n 3 gpurun_out/pytest_gpu.log
for v in 1 0; do WS_FUSEPP=$v timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/fpp_c2_$v.json 2>&1; done
for v in 1 0; do WS_FUSEPP=$v timeout 300 python bench.py --config c2 --precision f32 --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/fpp_c2f32_$v.json 2>&1; done
for v in 1 0; do WS_FUSEPP=$v timeout 600 python bench.py --config c5 --precision f32 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/fpp_c5f32_$v.json 2>&1; done
for v in 1 0; do WS_FUSEPP=$v timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/fpp_c5_$v.json 2>&1; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/fpp_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["value"]/1e9,3), d["ms_per_step"], d["roofline"].get("kernel_ms"), d["roofline"].get("speeds_kernel_ms"), d.get("simulation",{}).get("cell_updates_per_s",0)/1e9)
    except Exception as e: print(f, "ERR", open(f).read()[-400:])
PY
