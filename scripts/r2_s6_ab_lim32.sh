# one-select limiter ratio (WS_LIMSEL=1: vlim) on the two-wave fp32 kernels (policy: fp64 two-wave only)
. scripts/r2_s6_ab_fn.sh
for c in c4 c3; do for p in f32 f32fast; do for v in "" vlim; do ab lim_${c}_${p}_${v:-def} "$v" $c $p; done; done; done
export WAVESTEP_LIB=$PWD/paper_1308_1464_b200/_lib/vlim/libwavestep.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32fast.py -q -x > gpurun_out/ab8_lim_parity.log 2>&1; echo parity_rc=$?; tail -n 2 gpurun_out/ab8_lim_parity.log
