python tools/e2e_timeline.py > gpurun_out/e2e_tl.txt 2>&1; tail -3 gpurun_out/e2e_tl.txt
timeout 300 python -m pytest tests -m gpu -q -k "async or upload or order or download" > gpurun_out/pytest_e2e.log 2>&1; echo rc=$?; tail -n 2 gpurun_out/pytest_e2e.log
timeout 300 python bench.py --steps 20 --warmup 3 --cpu-seconds 2 > gpurun_out/bench_e2e.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_e2e.json').read().strip().splitlines()[-1]); print(d['value']/1e9, d['e2e'])"
