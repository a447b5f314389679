// ws_inst_acoustics_var.cu — kernel instantiations for the AcousticsVar plugin (fp64 + fp32,
// order 1 and the three limiters).  Compiled in parallel with the other
// ws_inst_*.cu units; see ws_host.cuh.
#include <cmath>

#include "ws_host.cuh"

namespace wsh {

Ops ops_acoustics_var(int prec, int order, int lim) {
  if (prec == WS_FP32_FAST) return ops_fast_acoustics_var(order, lim);
  return prec == WS_FP32 ? pick_lim<AcousticsVar, float>(order, lim) : pick_lim<AcousticsVar, double>(order, lim);
}

int riemann_acoustics_var(const double* p, int dir, long long n, const double* ql, const double* qr,
                   const double* al, const double* ar, double* w, double* s, double* am,
                   double* ap, int* codes) {
  (void)p;
  AcousticsVar::Params<double> P{0.0};
  return riemann_t<AcousticsVar>(P, dir, n, ql, qr, al, ar, w, s, am, ap, codes);
}

}  // namespace wsh
