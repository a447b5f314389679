# A/B: 3-component fp64 line kernel, 2 CTAs x 10 warps (default) vs persistent 1 CTA x 15 warps with cp.async prefetch
for cfg in c5 c4 c2 c1; do
  for p in 0 1; do
    WS_PERSIST3=$p python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu --no-ref-code > gpurun_out/p3_${cfg}_$p.json 2> gpurun_out/p3_${cfg}_$p.err
    python - gpurun_out/p3_${cfg}_$p.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(d['roofline']['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
PY
  done
done
WS_PERSIST3=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_recipes.py -q -x -k "second_order or many_tiles or c1 or c4_recipe or c5_fp64 or tiny or t_final" > gpurun_out/p3_pytest.log 2>&1; echo p3_pytest_rc=$?; tail -3 gpurun_out/p3_pytest.log
