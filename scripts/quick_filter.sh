# tile pre-pass: GPU tests, bench default vs edge filter vs exact pre-pass, CTA timeline
set -x
timeout 300 python -m pytest tests/test_gpu_cfl_filter.py -x -q > gpurun_out/pytest_filter.log 2>&1; echo pytest_rc=$?
for v in tile exact; do WS_SPEEDS=$v timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_$v.json 2>&1; echo rc=$?; done
for p in f64 f32; do timeout 600 python bench.py --config c5 --precision $p --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c5$p.json 2>&1; echo rc=$?; done
timeout 120 python tools/cta_trace.py --steps 100 --flush > gpurun_out/trace_c2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -n 3 gpurun_out/pytest_filter.log; tail -n 3 gpurun_out/pytest_gpu.log; cat gpurun_out/trace_c2.txt
python - <<'PY'
import json
for f in ["bench_tile","bench_exact","bench_c5f64","bench_c5f32"]:
    try:
        d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, d["value"]/1e9, d["ms_per_step"], d["roofline"].get("kernel_ms"), d["roofline"].get("speeds_kernel_ms"), d.get("simulation",{}).get("cell_updates_per_s"))
    except Exception as e: print(f, "ERR", e, open(f"gpurun_out/{f}.json").read()[-800:])
PY
