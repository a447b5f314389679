timeout 300 python -m pytest tests/test_gpu_cfl_filter.py -x -q > gpurun_out/pytest_filter.log 2>&1; echo pytest_rc=$?
for v in tile exact; do WS_SPEEDS=$v timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/exp_c2_$v.json 2>&1; done
for p in f64 f32; do timeout 600 python bench.py --config c5 --precision $p --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/exp_c5$p.json 2>&1; done
tail -n 2 gpurun_out/pytest_filter.log
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/exp_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["value"]/1e9,3), d["ms_per_step"], d["roofline"].get("kernel_ms"), d["roofline"].get("speeds_kernel_ms"), d["simulation"]["cell_updates_per_s"]/1e9)
    except Exception as e: print(f, "ERR", open(f).read()[-500:])
PY
timeout 120 python tools/cta_trace.py --steps 100 --flush > gpurun_out/trace_c2.txt 2>&1; head -5 gpurun_out/trace_c2.txt
