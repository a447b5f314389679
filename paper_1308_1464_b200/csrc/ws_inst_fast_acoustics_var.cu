// ws_inst_fast_acoustics_var.cu — the fp32 throughput mode (WS_FP32_FAST) of the
// AcousticsVar plugin: the same kernel templates instantiated for Fast<AcousticsVar>, compiled
// with --fmad=true -prec-div=false -prec-sqrt=false (build.py FAST_FLAGS).
#include "ws_host.cuh"

namespace wsh {

Ops ops_fast_acoustics_var(int order, int lim) { return pick_lim<Fast<AcousticsVar>, float>(order, lim); }

}  // namespace wsh
