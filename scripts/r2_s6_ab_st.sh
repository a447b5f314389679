# A/B of the non-inlined full-tile store (WS_FASTSTORE=1: vst) vs default, then parity on the variant
. scripts/r2_s6_ab_fn.sh
for c in c4 c5 c3 c2; do for v in "" vst; do ab st_${c}_f64_${v:-def} "$v" $c f64; done; done
for c in c4 c5; do for v in "" vst; do ab st_${c}_f32_${v:-def} "$v" $c f32; done; done
export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/vst/libwavestep.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_recipes.py tests/test_gpu_multishard.py tests/test_gpu_cfl_filter.py -q -x > gpurun_out/ab8_st_parity.log 2>&1; echo parity_rc=$?; tail -n 3 gpurun_out/ab8_st_parity.log
