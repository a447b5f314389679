# round 2: k_run_small (multi-step cooperative kernel) tests + full GPU suite,
# C1 line, C2 A/B (default / WS_PDL=0 / 2-CTA build)
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2s_pytest.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/r2s_pytest.log
python -c "import __graft_entry__ as g; g.smoke()"
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2s_c1.json 2> gpurun_out/r2s_c1.err; echo c1 rc=$?
WS_RUN_SMALL=0 timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2s_c1_nosmall.json 2> gpurun_out/r2s_c1_nosmall.err
for v in def nopdl lb2; do
  unset WAVESTEP_LIB WS_PDL
  [ $v = nopdl ] && export WS_PDL=0
  [ $v = lb2 ] && export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/lb2/libwavestep.so
  timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu --no-e2e --no-ref-code > gpurun_out/r2s_c2_$v.json 2> gpurun_out/r2s_c2_$v.err
done
unset WAVESTEP_LIB WS_PDL
for f in gpurun_out/r2s_c*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r=d['roofline']
    print(sys.argv[1], round(d['value']/1e9,3), 'G/s ms/step', round(d['ms_per_step']*1e3,1), 'us  update', round(r['kernel_ms']*1e3,1), 'speeds', round(r.get('speeds_kernel_ms',0)*1e3,1), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
done
