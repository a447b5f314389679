// ws_inst_fast_advection.cu — the fp32 throughput mode (WS_FP32_FAST) of the
// Advection plugin: the same kernel templates instantiated for Fast<Advection>, compiled
// with --fmad=true -prec-div=false -prec-sqrt=false (build.py FAST_FLAGS).
#include "ws_host.cuh"

namespace wsh {

Ops ops_fast_advection(int order, int lim) { return pick_lim<Fast<Advection>, float>(order, lim); }

}  // namespace wsh
