# A/B of ptxas --register-usage-level=2 (vru2; default level 5) on every config, then parity on the variant
. scripts/r2_s6_ab_fn.sh
for c in c5 c2 c4 c3 c1; do for v in "" vru2; do ab ru_${c}_f64_${v:-def} "$v" $c f64; done; done
for c in c5 c4 c3; do for p in f32 f32fast; do for v in "" vru2; do ab ru_${c}_${p}_${v:-def} "$v" $c $p; done; done; done
export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/vru2/libwavestep.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_recipes.py tests/test_gpu_multishard.py tests/test_gpu_cfl_filter.py tests/test_gpu_fp32fast.py tests/test_gpu_run_small.py -q -x > gpurun_out/ab8_ru_parity.log 2>&1; echo parity_rc=$?; tail -n 3 gpurun_out/ab8_ru_parity.log
