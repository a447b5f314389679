# final pass, part 2: the config lines after the per-precision ncu entries
for c in c3 c4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/fin_$c.json 2> gpurun_out/fin_$c.err; echo "$c rc=$?"
done
for c in c5 c4 c3; do for p in f32 f32fast; do
  timeout 900 python bench.py --config $c --precision $p --steps 10 --warmup 3 --no-cpu > gpurun_out/fin_${c}_$p.json 2> gpurun_out/fin_${c}_$p.err; echo "$c $p rc=$?"
done; done
for f in gpurun_out/fin_c3*.json gpurun_out/fin_c4*.json gpurun_out/fin_c5_*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d.get('roofline',{})
    print(sys.argv[1], round(d['value']/1e9,4), 'G/s', 'fp64', (r.get('fp64') or {}).get('frac'), 'issue', (r.get('issue') or {}).get('frac'), 'hbm', r.get('frac'))
except Exception as ex: print(sys.argv[1], 'FAILED', ex)
PY
done
