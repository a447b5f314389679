// ws_inst_advection.cu — kernel instantiations for the Advection plugin (fp64 +
// fp32, order 1 and the three limiters).  See ws_host.cuh.
#include <cmath>

#include "ws_host.cuh"

namespace wsh {

Ops ops_advection(int prec, int order, int lim) {
  if (prec == WS_FP32_FAST) return ops_fast_advection(order, lim);
  return prec == WS_FP32 ? pick_lim<Advection, float>(order, lim)
                         : pick_lim<Advection, double>(order, lim);
}

int riemann_advection(const double* p, int dir, long long n, const double* ql, const double* qr,
                      const double* al, const double* ar, double* w, double* s, double* am,
                      double* ap, int* codes) {
  Advection::Params<double> P{p[0], p[1]};
  return riemann_t<Advection>(P, dir, n, ql, qr, al, ar, w, s, am, ap, codes);
}

}  // namespace wsh
