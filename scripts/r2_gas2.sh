# A/B: 4-component fp64 line kernel at 2 x 10-warp CTAs per SM (WS_GAS2=1
# build) vs the default 15-warp persistent CTA (1 per SM): C3 (HLLE, minmod)
for v in def gas2; do
  if [ $v = gas2 ]; then export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/gas2/libwavestep.so; else unset WAVESTEP_LIB; fi
  timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --no-e2e --no-ref-code > gpurun_out/gas_c3_$v.json 2> gpurun_out/gas_c3_$v.err
  python - gpurun_out/gas_c3_$v.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(r['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
PY
done
export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/gas2/libwavestep.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_recipes.py -q -x -k "euler or c3" > gpurun_out/gas_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/gas_pytest.log
unset WAVESTEP_LIB
