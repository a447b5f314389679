# full GPU suite + smoke on the current default build; C4 A/B (3 vs 2 CTAs/SM)
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2u_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2u_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for v in def lb2; do
  if [ $v = lb2 ]; then export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/lb2/libwavestep.so; else unset WAVESTEP_LIB; fi
  timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-ref-code > gpurun_out/r2u_c4_$v.json 2> gpurun_out/r2u_c4_$v.err
  python - gpurun_out/r2u_c4_$v.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(r['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
PY
done
unset WAVESTEP_LIB
