// ws_inst_fast_acoustics_const.cu — the fp32 throughput mode (WS_FP32_FAST) of the
// AcousticsConst plugin: the same kernel templates instantiated for Fast<AcousticsConst>, compiled
// with --fmad=true -prec-div=false -prec-sqrt=false (build.py FAST_FLAGS).
#include "ws_host.cuh"

namespace wsh {

Ops ops_fast_acoustics_const(int order, int lim) { return pick_lim<Fast<AcousticsConst>, float>(order, lim); }

}  // namespace wsh
