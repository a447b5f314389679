# ws_step on small static-speed grids through k_run_small: suite + C1 lines
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/rs4_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/rs4_pytest.log
for v in 1 0; do
  WS_RUN_SMALL=$v timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/rs4_c1_$v.json 2> gpurun_out/rs4_c1_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/rs4_c1_$v.json').read().strip().splitlines()[-1]); print('WS_RUN_SMALL=$v', d['value']/1e9, d['ms_per_step'], d['simulation']['cell_updates_per_s']/1e9, d['gpu_launches'])"
done
