timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/st2_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/st2_pytest.log
for a in "--config c4" "--config c1" "--config c4 --strong --force-sharded"; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-ref-code $a > gpurun_out/st.json 2> gpurun_out/st.err; echo "[$a] rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/st.json').read().strip().splitlines()[-1]); print(' ', d['config']['workload'], round(d['value']/1e9,3), 'G/s', (d.get('simulation') or {}).get('cell_updates_per_s',0)/1e9)" || tail -5 gpurun_out/st.err
done
