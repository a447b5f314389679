// ws_inst_shallow_roe.cu — kernel instantiations for the ShallowRoe plugin (fp64 + fp32,
// order 1 and the three limiters).  Compiled in parallel with the other
// ws_inst_*.cu units; see ws_host.cuh.
#include <cmath>

#include "ws_host.cuh"

namespace wsh {

Ops ops_shallow_roe(int prec, int order, int lim) {
  if (prec == WS_FP32_FAST) return ops_fast_shallow_roe(order, lim);
  return prec == WS_FP32 ? pick_lim<ShallowRoe, float>(order, lim) : pick_lim<ShallowRoe, double>(order, lim);
}

int riemann_shallow_roe(const double* p, int dir, long long n, const double* ql, const double* qr,
                   const double* al, const double* ar, double* w, double* s, double* am,
                   double* ap, int* codes) {
  ShallowRoe::Params<double> P{p[0], std::sqrt(p[0])};
  return riemann_t<ShallowRoe>(P, dir, n, ql, qr, al, ar, w, s, am, ap, codes);
}

}  // namespace wsh
