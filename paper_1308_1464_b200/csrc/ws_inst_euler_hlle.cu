// ws_inst_euler_hlle.cu — kernel instantiations for the EulerHLLE plugin (fp64 + fp32,
// order 1 and the three limiters).  Compiled in parallel with the other
// ws_inst_*.cu units; see ws_host.cuh.
#include <cmath>

#include "ws_host.cuh"

namespace wsh {

Ops ops_euler_hlle(int prec, int order, int lim) {
  if (prec == WS_FP32_FAST) return ops_fast_euler_hlle(order, lim);
  return prec == WS_FP32 ? pick_lim<EulerHLLE, float>(order, lim) : pick_lim<EulerHLLE, double>(order, lim);
}

int riemann_euler_hlle(const double* p, int dir, long long n, const double* ql, const double* qr,
                   const double* al, const double* ar, double* w, double* s, double* am,
                   double* ap, int* codes) {
  EulerHLLE::Params<double> P{p[0] - 1.0, p[0]};
  return riemann_t<EulerHLLE>(P, dir, n, ql, qr, al, ar, w, s, am, ap, codes);
}

}  // namespace wsh
