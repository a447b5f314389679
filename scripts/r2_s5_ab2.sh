# A/B of the per-solver line-kernel policy (default) vs all-at-once staging (vsb0) and batches of 2 for every solver (vsb2); then the GPU suite on the default
ab() {
  if [ -n "$2" ]; then export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/$2/libwavestep.so; else unset WAVESTEP_LIB; fi
  timeout 600 python bench.py --config $3 --precision $4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-ref-code > gpurun_out/ab6_$1.json 2> gpurun_out/ab6_$1.err
  python - gpurun_out/ab6_$1.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], round(d['value']/1e9,3), 'G/s  update ms', round(r['kernel_ms'],4), 'sim', round(d['simulation']['cell_updates_per_s']/1e9,3))
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
}
for c in c4 c5 c2 c3 c1; do for v in "" vsb0 vsb2; do ab ${c}_f64_${v:-def} "$v" $c f64; done; done
for c in c4 c5; do for v in "" vsb2; do ab ${c}_f32_${v:-def} "$v" $c f32; done; done
unset WAVESTEP_LIB
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/ab6_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/ab6_pytest.log
