# the scale.sh configurations at world size 1 (forced row-strip path)
for a in "--config c5 --strong" "--config c3 --strong" "--config c4 --strong" "--device-halo" "--config c3 --strong --device-reduce"; do
  timeout 900 python bench.py --force-sharded --steps 10 --warmup 3 --no-e2e $a > gpurun_out/s1.json 2> gpurun_out/s1.err; echo "[$a] rc=$?"
  python - <<'PY'
import json
try:
    d=json.loads(open('gpurun_out/s1.json').read().strip().splitlines()[-1])
    print(' ', d['config']['workload'], round(d['value']/1e9,3), 'G/s', d['measurement'].get('issue'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))
except Exception as e:
    print('  FAILED', e); print(open('gpurun_out/s1.err').read()[-1500:])
PY
done
