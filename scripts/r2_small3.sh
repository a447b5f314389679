# k_run_small with neighbour waits and a lagged global check: phases, tests, C1 line
WAVESTEP_LIB=paper_1308_1464_b200/_lib/rsprof/libwavestep.so timeout 120 python tools/run_small_phases.py --steps 40 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_run_small.py tests/test_gpu_recipes.py tests/test_gpu_checked.py -k "run_small or c1 or checked" -q -x > gpurun_out/rs3_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/rs3_pytest.log
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/rs3_c1.json 2> gpurun_out/rs3_c1.err; echo c1 rc=$?
python -c "import json; d=json.loads(open('gpurun_out/rs3_c1.json').read().strip().splitlines()[-1]); print(d['value']/1e9, d['simulation'])"
