// ws_inst_acoustics_const.cu — kernel instantiations for the AcousticsConst plugin (fp64 + fp32,
// order 1 and the three limiters).  Compiled in parallel with the other
// ws_inst_*.cu units; see ws_host.cuh.
#include <cmath>

#include "ws_host.cuh"

namespace wsh {

Ops ops_acoustics_const(int prec, int order, int lim) {
  if (prec == WS_FP32_FAST) return ops_fast_acoustics_const(order, lim);
  return prec == WS_FP32 ? pick_lim<AcousticsConst, float>(order, lim) : pick_lim<AcousticsConst, double>(order, lim);
}

int riemann_acoustics_const(const double* p, int dir, long long n, const double* ql, const double* qr,
                   const double* al, const double* ar, double* w, double* s, double* am,
                   double* ap, int* codes) {
  double c = std::sqrt(p[1] / p[0]), z = p[0] * c;
  AcousticsConst::Params<double> P{z, 2.0 * z, c};
  return riemann_t<AcousticsConst>(P, dir, n, ql, qr, al, ar, w, s, am, ap, codes);
}

}  // namespace wsh
