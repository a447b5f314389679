// ws_inst_shallow_roe.cu — kernel instantiations for the ShallowRoe plugin (fp64; fp32 in
// ws_inst_f32_shallow_roe.cu), order 1 and the three limiters.  Compiled in parallel with the
// other ws_inst_*.cu units; see ws_host.cuh.  This unit alone is compiled with ptxas
// --register-usage-level=2 (build.py UNIT_FLAGS): the three-wave fp64 line kernel then keeps
// 8 instead of 68 bytes of spills at its 64-register cap (C5 +4 %, C2 +5 %); every other
// kernel is equal or slower with it (profiles/r2_s6_ab.md).
#include <cmath>

#include "ws_host.cuh"

namespace wsh {

Ops ops_shallow_roe(int prec, int order, int lim) {
  if (prec == WS_FP32_FAST) return ops_fast_shallow_roe(order, lim);
  return prec == WS_FP32 ? ops_f32_shallow_roe(order, lim) : pick_lim<ShallowRoe, double>(order, lim);
}

int riemann_shallow_roe(const double* p, int dir, long long n, const double* ql, const double* qr,
                   const double* al, const double* ar, double* w, double* s, double* am,
                   double* ap, int* codes) {
  ShallowRoe::Params<double> P{p[0], std::sqrt(p[0])};
  return riemann_t<ShallowRoe>(P, dir, n, ql, qr, al, ar, w, s, am, ap, codes);
}

}  // namespace wsh
