for cfg in c5 c4 c2; do
  for p in 0 1; do
    WS_PERSIST3=$p python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu --no-ref-code > gpurun_out/p3b_${cfg}_$p.json 2> gpurun_out/p3b_${cfg}_$p.err
    python - gpurun_out/p3b_${cfg}_$p.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(d['roofline']['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
  done
done
WS_PERSIST3=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "second_order or many_tiles or tiny or t_final or persistent" > gpurun_out/p3b_pytest.log 2>&1; echo p3_pytest_rc=$?; tail -2 gpurun_out/p3b_pytest.log
bash scripts/r2_sanitize.sh
