# round 2 evidence: headline bench (both arms, driver flags), secondary config
# lines, the reference-format bench matrix (drop-in driver.step rows)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err; echo ref_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/ev_c5.json 2> gpurun_out/ev_c5.err; echo c5_rc=$?
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/ev_$c.json 2> gpurun_out/ev_$c.err; echo "$c rc=$?"
done
for p in f32 f32fast; do
  timeout 900 python bench.py --config c5 --precision $p --steps 10 --warmup 3 --no-cpu > gpurun_out/ev_c5_$p.json 2> gpurun_out/ev_c5_$p.err; echo "c5 $p rc=$?"
done
bash scripts/matrix.sh
for f in gpurun_out/ev_*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d.get('roofline',{})
    e=d.get('e2e') or {}
    print(sys.argv[1], round(d['value']/1e9,4), 'G/s  ms/step', round(d['ms_per_step'],4), 'e2e', round((e.get('value') or 0)/1e9,3), 'sim', round((d.get('simulation') or {}).get('cell_updates_per_s',0)/1e9,3), 'cpu', (d.get('cpu_baseline') or {}).get('value'))
except Exception as ex: print(sys.argv[1], 'FAILED', ex)
PY
done
