# static-speed shards: tile pre-pass (bad-cell tiles only); suites + C4 strong at world 1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/st_pytest.log 2>&1; echo pytest_rc=$?; tail -15 gpurun_out/st_pytest.log | grep -v "^\.\.\." | tail -8
for a in "--config c4 --strong" "--config c1 --strong"; do
  timeout 900 python bench.py --force-sharded --steps 10 --warmup 3 --no-e2e --no-cpu $a > gpurun_out/st.json 2> gpurun_out/st.err; echo "[$a] rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/st.json').read().strip().splitlines()[-1]); print(' ', d['config']['workload'], round(d['value']/1e9,3), 'G/s')" || tail -5 gpurun_out/st.err
done
