# A/B of the non-inlined interior staging (WS_FASTSTAGE=1: vfs) vs default, then parity on the variant
. scripts/r2_s6_ab_fn.sh
for c in c4 c5 c3 c2; do for v in "" ${VARIANTS:-vfs}; do ab fs_${c}_f64_${v:-def} "$v" $c f64; done; done
for c in c4 c5; do for v in "" ${VARIANTS:-vfs}; do ab fs_${c}_f32_${v:-def} "$v" $c f32; done; done
export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/${PARITY_VARIANT:-vfs}/libwavestep.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_recipes.py tests/test_gpu_multishard.py -q -x > gpurun_out/ab8_fs_parity.log 2>&1; echo parity_rc=$?; tail -n 3 gpurun_out/ab8_fs_parity.log
