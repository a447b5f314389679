// ws_inst_fast_shallow_roe.cu — the fp32 throughput mode (WS_FP32_FAST) of the
// ShallowRoe plugin: the same kernel templates instantiated for Fast<ShallowRoe>, compiled
// with --fmad=true -prec-div=false -prec-sqrt=false (build.py FAST_FLAGS).
#include "ws_host.cuh"

namespace wsh {

Ops ops_fast_shallow_roe(int order, int lim) { return pick_lim<Fast<ShallowRoe>, float>(order, lim); }

}  // namespace wsh
