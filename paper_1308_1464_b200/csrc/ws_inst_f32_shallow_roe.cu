// ws_inst_f32_shallow_roe.cu — the fp32 kernels of the ShallowRoe plugin (bitwise vs the fp32
// oracle; the throughput mode is ws_inst_fast_shallow_roe.cu).  A unit of its own because the
// fp64 unit is compiled with a ptxas option that costs the fp32 kernels 1-3 % (build.py
// UNIT_FLAGS).
#include "ws_host.cuh"

namespace wsh {

Ops ops_f32_shallow_roe(int order, int lim) { return pick_lim<ShallowRoe, float>(order, lim); }

}  // namespace wsh
