# quick check of a kernel change: parity subset on the default build, then one bench line per config
unset WAVESTEP_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_recipes.py tests/test_gpu_multishard.py tests/test_gpu_checked.py -q -x > gpurun_out/s6q_parity.log 2>&1; echo parity_rc=$?; tail -n 2 gpurun_out/s6q_parity.log
. scripts/r2_s6_ab_fn.sh
for c in c4 c5 c3 c2; do ab q_${c}_f64 "" $c f64; done
for c in c4 c5; do ab q_${c}_f32 "" $c f32; done
