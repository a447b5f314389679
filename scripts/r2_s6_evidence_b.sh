# round-2 final evidence (v5), part B (after profiles/ncu_traffic.json was refreshed from part A):
# smoke, the GPU suite, both arms of the headline, every config line (fp64, fp32, f32fast), the bench matrix
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v5_smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/v5_pytest_gpu.log 2>&1; echo pytest_rc=$?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/v5_ref.json 2> gpurun_out/v5_ref.err; echo ref_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/v5_c5.json 2> gpurun_out/v5_c5.err; echo c5_rc=$?
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/v5_$c.json 2> gpurun_out/v5_$c.err; echo "$c rc=$?"
done
for c in c5 c4 c3; do for p in f32 f32fast; do
  timeout 900 python bench.py --config $c --precision $p --steps 10 --warmup 3 --no-cpu > gpurun_out/v5_${c}_$p.json 2> gpurun_out/v5_${c}_$p.err; echo "$c $p rc=$?"
done; done
bash scripts/matrix.sh
set +x
tail -n 3 gpurun_out/v5_smoke.log gpurun_out/v5_pytest_gpu.log
for f in gpurun_out/v5_*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d.get('roofline',{})
    e=d.get('e2e') or {}
    print(sys.argv[1], round(d['value']/1e9,4), 'G/s  ms/step', round(d['ms_per_step'],4), 'e2e', round((e.get('value') or 0)/1e9,3), 'sim', round((d.get('simulation') or {}).get('cell_updates_per_s',0)/1e9,3), 'hbm', r.get('frac'), 'fp64', (r.get('fp64') or {}).get('frac'), 'issue', (r.get('issue') or {}).get('frac'))
except Exception as ex: print(sys.argv[1], 'FAILED', ex)
PY
done
