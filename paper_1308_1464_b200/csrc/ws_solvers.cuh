// ws_solvers.cuh — pointwise Riemann solvers as parallelism-unaware device
// plugins (the paper's decoupling goal; reference plugin
// contract: class Kernel, kernels.py:374-393).
//
// A solver is a struct with
//   NEQ, NW, NAUX, NPR           components, waves, aux fields, per-cell primitives
//   STATIC_SPEEDS                speeds independent of q (acoustics)
//   Params<R>                    bound parameters (reference make_kernel, kernels.py:396-440)
//   prims<M>(q, aux, P, pr, ok)  per-cell quantities shared by the 4 edges of a cell
//   solve<NI,M>(ql,qr,pl,pr,al,ar,P,W,s,amdq,apdq,ok)  one edge, NI = normal slot (1=x, 2=y)
//   probe<NI,M>(...,smax,ok) -> code  admissibility tests in the reference order and
//                                the edge's max |s| (for the CFL reduction)
//   cell_ok / probe_fast         the per-cell part of those tests / the rest
// M is the math policy for / and sqrt (ws_math.cuh): IeeeMath, or FastMath
// whose results equal IeeeMath's whenever `ok` stays true (callers
// re-evaluate with IeeeMath otherwise).
// Every expression keeps the association of the numpy oracle
// (oracle/wavestep_oracle.py) and of the reference for the solvers it has;
// the translation unit is compiled with --fmad=false, IEEE div/sqrt, so
// fp64 results are bitwise identical to numpy.
#pragma once
#include <climits>
#include "ws_common.cuh"
#include "ws_math.cuh"

namespace ws {

constexpr double FLOOR = 1e-300;  // reference ADMISSIBILITY_FLOOR, kernels.py:34

// code = (stage + 1) | (component << 8); 0 = admissible
template <class R, int N>
__device__ __forceinline__ int finite_code(const R* ql, const R* qr) {
#pragma unroll
  for (int m = 0; m < N; ++m)
    if (!isfinite(ql[m])) return 1 | (m << 8);
#pragma unroll
  for (int m = 0; m < N; ++m)
    if (!isfinite(qr[m])) return 2 | (m << 8);
  return 0;
}

// exponent-field test, no FP64 pipe work
template <class R, int N> __device__ __forceinline__ bool all_finite(const R* q) {
  bool ok = true;
#pragma unroll
  for (int m = 0; m < N; ++m) ok = ok && isfinite(q[m]);
  return ok;
}

// float32: every positive float exceeds 1e-300, so the floor is 0 (numpy's
// float32 comparison against 1e-300 behaves the same way)
template <class R> __device__ __forceinline__ R floor_v() { return (R)0; }
template <> __device__ __forceinline__ double floor_v<double>() { return FLOOR; }
template <class R> __device__ __forceinline__ bool bad_pos(R v) { return !(v > floor_v<R>()); }

// ---------------------------------------------------------------------------
// constant-coefficient acoustics — reference kernels.py:181-213
struct AcousticsConst {
  static constexpr int NEQ = 3, NW = 2, NAUX = 0, NPR = 0;
  static constexpr bool STATIC_SPEEDS = true;
  // Tile form for row-strip shards (k_speeds_t): the speeds are static, so a
  // tile only needs probing if one of its new cells is inadmissible (then
  // the checked probe finds the reference-order first interface); a[0] =
  // "some cell is not finite" over the tile.  Aux is static: the first
  // pre-pass after an upload probes every tile.
  static constexpr bool HAS_TILE = true;
  static constexpr int NACC = 4;
  static constexpr unsigned ACC_MIN = 0x0u;
  __device__ static __forceinline__ void acc_init(int (&a)[NACC]) {
    a[0] = 0; a[1] = 0; a[2] = 0; a[3] = 0;
  }
  template <class R, class P>
  __device__ static __forceinline__ void tile_acc(const R* q, const P&, int (&a)[NACC]) {
    a[0] = max(a[0], all_finite<R, NEQ>(q) ? 0 : 1);
  }
  template <class R, class P>
  __device__ static __forceinline__ void tile_bound(const int (&a)[NACC], const P&, R& bndx,
                                                    R& bndy) {
    bndx = bndy = a[0] ? (R)INFINITY : (R)0;
  }
  // structurally zero wave components (skipped by the limiter; adding the
  // oracle's exact zeros would not change any value)
  template <int NI> __host__ __device__ static constexpr bool wzero(int, int m) { return m == 3 - NI; }
  template <class R> struct Params { R z, twoz, c; };

  template <class M, class R, class P>
  __device__ static __forceinline__ void prims(const R*, const R*, const P&, R*, bool&) {}

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ void solve(const R* ql, const R* qr, const R*, const R*,
                                               const R*, const R*, const P& p, R (&W)[NW][NEQ],
                                               R (&s)[NW], R (&am)[NEQ], R (&ap)[NEQ],
                                               bool& ok) {
    constexpr int TI = 3 - NI;
    R dp = qr[0] - ql[0];
    R dn = qr[NI] - ql[NI];
    R a1 = M::div(-dp + p.z * dn, p.twoz, ok);
    R a2 = M::div(dp + p.z * dn, p.twoz, ok);
    W[0][0] = (-p.z) * a1; W[0][NI] = a1; W[0][TI] = (R)0;
    W[1][0] = p.z * a2;    W[1][NI] = a2; W[1][TI] = (R)0;
    s[0] = -p.c; s[1] = p.c;
#pragma unroll
    for (int m = 0; m < NEQ; ++m) { am[m] = (-p.c) * W[0][m]; ap[m] = p.c * W[1][m]; }
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ int probe(const R* ql, const R* qr, const R*, const R*,
                                              const R*, const R*, const P& p, R& smax, bool&) {
    smax = p.c;
    return finite_code<R, NEQ>(ql, qr);
  }

  // per-cell part of the admissibility tests; probe_fast assumes both cells pass
  template <class R, class P>
  __device__ static __forceinline__ bool cell_ok(const R* q, const R*, const R*, const P&) {
    return all_finite<R, NEQ>(q);
  }
  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ int probe_fast(const R*, const R*, const R*, const R*,
                                                   const R*, const R*, const P& p, R& smax,
                                                   bool&) {
    smax = p.c;
    return 0;
  }
};

// ---------------------------------------------------------------------------
// variable-coefficient acoustics, aux = (rho, c) — reference kernels.py:216-261
struct AcousticsVar {
  static constexpr int NEQ = 3, NW = 2, NAUX = 2, NPR = 1;  // pr[0] = Z = rho*c
  static constexpr bool STATIC_SPEEDS = true;
  // Tile form for row-strip shards (k_speeds_t): the speeds are static, so a
  // tile only needs probing if one of its new cells is inadmissible (then
  // the checked probe finds the reference-order first interface); a[0] =
  // "some cell is not finite" over the tile.  Aux is static: the first
  // pre-pass after an upload probes every tile.
  static constexpr bool HAS_TILE = true;
  static constexpr int NACC = 4;
  static constexpr unsigned ACC_MIN = 0x0u;
  __device__ static __forceinline__ void acc_init(int (&a)[NACC]) {
    a[0] = 0; a[1] = 0; a[2] = 0; a[3] = 0;
  }
  template <class R, class P>
  __device__ static __forceinline__ void tile_acc(const R* q, const P&, int (&a)[NACC]) {
    a[0] = max(a[0], all_finite<R, NEQ>(q) ? 0 : 1);
  }
  template <class R, class P>
  __device__ static __forceinline__ void tile_bound(const int (&a)[NACC], const P&, R& bndx,
                                                    R& bndy) {
    bndx = bndy = a[0] ? (R)INFINITY : (R)0;
  }
  template <int NI> __host__ __device__ static constexpr bool wzero(int, int m) { return m == 3 - NI; }
  template <class R> struct Params { R unused; };

  template <class M, class R, class P>
  __device__ static __forceinline__ void prims(const R*, const R* a, const P&, R* pr, bool&) {
    pr[0] = a[0] * a[1];
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ void solve(const R* ql, const R* qr, const R* pl, const R* pr,
                                               const R* al, const R* ar, const P&, R (&W)[NW][NEQ],
                                               R (&s)[NW], R (&am)[NEQ], R (&ap)[NEQ],
                                               bool& ok) {
    constexpr int TI = 3 - NI;
    R zl = pl[0], zr = pr[0];
    R cl = al[1], cr = ar[1];
    R dp = qr[0] - ql[0];
    R dn = qr[NI] - ql[NI];
    R den = zl + zr;
    R a1 = M::div(-dp + zr * dn, den, ok);
    R a2 = M::div(dp + zl * dn, den, ok);
    W[0][0] = (-zl) * a1; W[0][NI] = a1; W[0][TI] = (R)0;
    W[1][0] = zr * a2;    W[1][NI] = a2; W[1][TI] = (R)0;
    s[0] = -cl; s[1] = cr;
#pragma unroll
    for (int m = 0; m < NEQ; ++m) { am[m] = (-cl) * W[0][m]; ap[m] = cr * W[1][m]; }
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ int probe(const R* ql, const R* qr, const R*, const R*,
                                              const R* al, const R* ar, const P&, R& smax,
                                              bool&) {
    smax = nmax(al[1], ar[1]);
    int c = finite_code<R, NEQ>(ql, qr);
    if (c) return c;
    // kernels.py:235-237: per side density then sound speed, left first
    if (bad_pos(al[0])) return 3;
    if (bad_pos(al[1])) return 4;
    if (bad_pos(ar[0])) return 5;
    if (bad_pos(ar[1])) return 6;
    return 0;
  }

  template <class R, class P>
  __device__ static __forceinline__ bool cell_ok(const R* q, const R* a, const R*, const P&) {
    return all_finite<R, NEQ>(q) && !bad_pos(a[0]) && !bad_pos(a[1]);
  }
  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ int probe_fast(const R*, const R*, const R*, const R*,
                                                   const R* al, const R* ar, const P&, R& smax,
                                                   bool&) {
    smax = nmax(al[1], ar[1]);
    return 0;
  }
};

// ---------------------------------------------------------------------------
// ideal gas, shared per-cell primitives (reference rp_euler u_l, p_l, sq_l: kernels.py:282-285, 289, 294)
//   pr = {u = q1/rho, v = q2/rho, p, sqrt(rho), sqrt(rho)*(E+p)/rho [, c]}
// p uses (u*u + v*v); the y sweep's (v*v + u*u) is the same IEEE sum.
template <class M, class R, class P>
__device__ __forceinline__ void gas_prims(const R* q, const P& p, R* pr, bool& ok) {
  R rho = q[0];
  R u = M::div(q[1], rho, ok);
  R v = M::div(q[2], rho, ok);
  R pp = p.gm1 * (q[3] - (R)0.5 * rho * (u * u + v * v));
  R sq = M::sqrt_(rho, ok);
  pr[0] = u; pr[1] = v; pr[2] = pp; pr[3] = sq; pr[4] = M::div(sq * (q[3] + pp), rho, ok);
}

// ---------------------------------------------------------------------------
// Tile accumulators of the ideal-gas solvers (k_update_w epilogue ->
// k_speeds_t).  Per new cell, from the approximate reciprocal seed of rho:
// u, v and c^2 = gamma (gamma-1) (E - |m|^2 / (2 rho)) / rho, plus a "safe"
// flag: finite, rho and E inside the seeds' range, internal energy at least
// KAPPA E (Mach ~< 40 in fp64, ~< 6 in fp32), so the approximations are
// accurate to 2^-8 and the exact path can neither find p <= floor nor lose
// Roe's c^2 > 0 to rounding.  Accumulators (sortable integer keys of the high
// words): max u, min u, max v, min v, max c^2, min c^2, min safe.
// Bound: with w the Roe weight, c_hat^2 = w c_l^2 + (1-w) c_r^2 + (gamma-1)/2
// w (1-w) |u_l - u_r|^2 <= max c^2 + (gamma-1)/8 |du|^2, and |u_hat| <= max
// |u|, so every HLLE / Roe edge speed of the folded tiles is at most
// max|u_n| + sqrt(max c^2 + (gamma-1)/8 (du^2 + dv^2)).
struct GasTile {
  static constexpr int NACC = 8;
  static constexpr unsigned ACC_MIN = 0x6Au;   // slots 1, 3, 5, 6
  __device__ static __forceinline__ int skey(int w) { return w ^ ((w >> 31) & 0x7fffffff); }
  template <class R> __device__ static __forceinline__ R ub_s(int k) {
    const int w = skey(k);
    return k >= 0 ? BoundMath::ub<R>(w) : BoundMath::lb<R>(w);
  }
  template <class R> __device__ static __forceinline__ R lb_s(int k) {
    const int w = skey(k);
    return k >= 0 ? BoundMath::lb<R>(w) : BoundMath::ub<R>(w);
  }
  __device__ static __forceinline__ void acc_init(int (&a)[NACC]) {
    a[0] = INT_MIN; a[1] = INT_MAX; a[2] = INT_MIN; a[3] = INT_MAX;
    a[4] = INT_MIN; a[5] = INT_MAX; a[6] = INT_MAX; a[7] = 0;
  }
  // gg2 = gamma (gamma-1) / 2: c^2 ~ gg2 (2E - m.u) / rho.  Bound-only
  // arithmetic (explicit FMAs; the parity-relevant code has none).
  template <class R>
  __device__ static __forceinline__ void acc(const R* q, R gg2, int (&a)[NACC]) {
    // internal energy >= KAPPA E as an exponent test: 2E - m.u >= 2^-KB (2E)
    constexpr int KB = sizeof(R) == 8 ? 9 : 3;
    constexpr int ESH = sizeof(R) == 8 ? 20 : 23;
    const int elo = sizeof(R) == 8 ? 0x07B00000 : 0x21800000;
    const R rho = q[0], mx = q[1], my = q[2], E = q[3];
    const R r = BoundMath::rcp(rho);
    const R u = mx * r, v = my * r;
    const R ei2 = fma((R)2, E, -fma(mx, u, my * v));   // 2 x internal energy density
    const R c2 = gg2 * ei2 * r;
    const int he = BoundMath::hw(E), hi2 = BoundMath::hw(ei2);
    const bool safe = BoundMath::pos_ok(rho) && BoundMath::abs_ok(mx) && BoundMath::abs_ok(my) &&
                      he >= elo && he < BoundMath::hw_hi<R>() &&
                      hi2 >= he - (KB << ESH) && hi2 > 0 &&
                      BoundMath::small(fabs(u)) && BoundMath::small(fabs(v)) && BoundMath::small(c2);
    const int ku = skey(BoundMath::hw(u)), kv = skey(BoundMath::hw(v));
    const int kc = BoundMath::hw(c2);
    a[0] = max(a[0], ku); a[1] = min(a[1], ku);
    a[2] = max(a[2], kv); a[3] = min(a[3], kv);
    a[4] = max(a[4], kc); a[5] = min(a[5], kc);
    a[6] = min(a[6], safe ? 1 : 0);
  }
  template <class R>
  __device__ static __forceinline__ void bound(const int (&a)[NACC], R gm1, R& bndx, R& bndy) {
    bndx = bndy = (R)INFINITY;
    if (a[6] < 1 || !(gm1 >= (R)(1.0 / 1048576.0))) return;
    const R umax = ub_s<R>(a[0]), umin = lb_s<R>(a[1]);
    const R vmax = ub_s<R>(a[2]), vmin = lb_s<R>(a[3]);
    const R c2u = BoundMath::ub<R>(a[4]) * (R)(1.0 + 1.0 / 64.0);
    const R c2l = BoundMath::lb<R>(a[5]) * (R)(1.0 - 1.0 / 64.0);
    const R au = nmax(fabs(umax), fabs(umin)), av = nmax(fabs(vmax), fabs(vmin));
    const R du = (umax - umin) + (fabs(umax) + fabs(umin)) * (R)(1.0 / 65536.0);
    const R dv = (vmax - vmin) + (fabs(vmax) + fabs(vmin)) * (R)(1.0 / 65536.0);
    const R ch2 = c2u + gm1 * (R)0.125 * (du * du + dv * dv);
    const R tol = sizeof(R) == 8 ? (R)(1.0 / 1099511627776.0) : (R)(1.0 / 16384.0);
    if (!(c2l > tol * (c2u + au * au + av * av))) return;
    const R ch = sqrt(ch2);
    const R bx = au + ch, by = av + ch;
    if (!(BoundMath::small(bx) && BoundMath::small(by))) return;
    bndx = bx; bndy = by;
  }
};

// Euler, Roe linearisation, no entropy fix — reference kernels.py:264-340
struct EulerRoe {
  static constexpr int NEQ = 4, NW = 3, NAUX = 0, NPR = 5;
  static constexpr bool STATIC_SPEEDS = false;
  // tile-filtered CFL pre-pass (GasTile)
  static constexpr bool HAS_TILE = true;
  static constexpr int NACC = GasTile::NACC;
  static constexpr unsigned ACC_MIN = GasTile::ACC_MIN;
  __device__ static __forceinline__ void acc_init(int (&a)[NACC]) { GasTile::acc_init(a); }
  template <class R, class P>
  __device__ static __forceinline__ void tile_acc(const R* q, const P& p, int (&a)[NACC]) {
    GasTile::acc(q, (R)0.5 * (p.gm1 + (R)1) * p.gm1, a);
  }
  template <class R, class P>
  __device__ static __forceinline__ void tile_bound(const int (&a)[NACC], const P& p, R& bx, R& by) {
    GasTile::bound(a, p.gm1, bx, by);
  }
  template <int NI> __host__ __device__ static constexpr bool wzero(int, int) { return false; }
  template <class R> struct Params { R gm1; };

  template <class M, class R, class P>
  __device__ static __forceinline__ void prims(const R* q, const R*, const P& p, R* pr, bool& ok) {
    gas_prims<M>(q, p, pr, ok);
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ void roe(const R* pl, const R* pr, const P& p, R& uh, R& vh,
                                             R& hh, R& kin, R& c2, bool& ok) {
    constexpr int UN = NI - 1, UT = 2 - NI;
    R ws = pl[3] + pr[3];
    uh = M::div(pl[3] * pl[UN] + pr[3] * pr[UN], ws, ok);
    vh = M::div(pl[3] * pl[UT] + pr[3] * pr[UT], ws, ok);
    hh = M::div(pl[4] + pr[4], ws, ok);
    kin = (R)0.5 * (uh * uh + vh * vh);
    c2 = p.gm1 * (hh - kin);
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ void solve(const R* ql, const R* qr, const R* pl, const R* pr,
                                               const R*, const R*, const P& p, R (&W)[NW][NEQ],
                                               R (&s)[NW], R (&am)[NEQ], R (&ap)[NEQ],
                                               bool& ok) {
    constexpr int TI = 3 - NI;
    R uh, vh, hh, kin, c2;
    roe<NI, M>(pl, pr, p, uh, vh, hh, kin, c2, ok);
    R ch = M::sqrt_(c2, ok);
    R d0 = qr[0] - ql[0];
    R dm = qr[NI] - ql[NI];
    R dt = qr[TI] - ql[TI];
    R de = qr[3] - ql[3];
    R ash = dt - vh * d0;
    R amid = M::div(p.gm1, c2, ok) * ((hh - uh * uh) * d0 + uh * dm - (de - ash * vh));
    R span = M::div(dm - uh * d0, ch, ok);
    R apl = (R)0.5 * (span + d0 - amid);
    R ami = d0 - amid - apl;
    W[0][0] = ami;  W[0][NI] = ami * (uh - ch);  W[0][TI] = ami * vh;       W[0][3] = ami * (hh - uh * ch);
    W[1][0] = amid; W[1][NI] = amid * uh;        W[1][TI] = amid * vh + ash; W[1][3] = amid * kin + ash * vh;
    W[2][0] = apl;  W[2][NI] = apl * (uh + ch);  W[2][TI] = apl * vh;       W[2][3] = apl * (hh + uh * ch);
    s[0] = uh - ch; s[1] = uh; s[2] = uh + ch;
    R n0 = nmin(s[0], (R)0), n1 = nmin(s[1], (R)0), n2 = nmin(s[2], (R)0);
    R p0 = nmax(s[0], (R)0), p1 = nmax(s[1], (R)0), p2 = nmax(s[2], (R)0);
#pragma unroll
    for (int m = 0; m < NEQ; ++m) {
      am[m] = n0 * W[0][m] + n1 * W[1][m] + n2 * W[2][m];
      ap[m] = p0 * W[0][m] + p1 * W[1][m] + p2 * W[2][m];
    }
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ int probe(const R* ql, const R* qr, const R* pl, const R* pr,
                                              const R*, const R*, const P& p, R& smax, bool& ok) {
    int c = finite_code<R, NEQ>(ql, qr);
    if (c) { smax = (R)0; return c; }
    if (bad_pos(ql[0])) { smax = (R)0; return 3; }
    if (bad_pos(qr[0])) { smax = (R)0; return 4; }
    if (bad_pos(pl[2])) { smax = (R)0; return 5; }
    if (bad_pos(pr[2])) { smax = (R)0; return 6; }
    return probe_fast<NI, M>(ql, qr, pl, pr, (const R*)nullptr, (const R*)nullptr, p, smax, ok);
  }

  template <class R, class P>
  __device__ static __forceinline__ bool cell_ok(const R* q, const R*, const R* pr, const P&) {
    return all_finite<R, NEQ>(q) && !bad_pos(q[0]) && !bad_pos(pr[2]);
  }
  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ int probe_fast(const R*, const R*, const R* pl, const R* pr,
                                                   const R*, const R*, const P& p, R& smax,
                                                   bool& ok) {
    R uh, vh, hh, kin, c2;
    roe<NI, M>(pl, pr, p, uh, vh, hh, kin, c2, ok);
    if (!(c2 > (R)0)) { smax = (R)0; return 7; }
    R ch = M::sqrt_(c2, ok);
    // |uh| never exceeds max(|uh-c|, |uh+c|) for c >= 0 (rounding is monotone)
    smax = nmax(fabs(uh - ch), fabs(uh + ch));
    return 0;
  }
};

// Euler HLLE (builder-owned formula; oracle rp_euler_hlle)
struct EulerHLLE {
  static constexpr int NEQ = 4, NW = 2, NAUX = 0, NPR = 6;  // gas prims + c
  static constexpr bool STATIC_SPEEDS = false;
  // tile-filtered CFL pre-pass (GasTile)
  static constexpr bool HAS_TILE = true;
  static constexpr int NACC = GasTile::NACC;
  static constexpr unsigned ACC_MIN = GasTile::ACC_MIN;
  __device__ static __forceinline__ void acc_init(int (&a)[NACC]) { GasTile::acc_init(a); }
  template <class R, class P>
  __device__ static __forceinline__ void tile_acc(const R* q, const P& p, int (&a)[NACC]) {
    GasTile::acc(q, (R)0.5 * p.gam * p.gm1, a);
  }
  template <class R, class P>
  __device__ static __forceinline__ void tile_bound(const int (&a)[NACC], const P& p, R& bx, R& by) {
    GasTile::bound(a, p.gm1, bx, by);
  }
  template <int NI> __host__ __device__ static constexpr bool wzero(int, int) { return false; }
  template <class R> struct Params { R gm1, gam; };

  template <class M, class R, class P>
  __device__ static __forceinline__ void prims(const R* q, const R*, const P& p, R* pr, bool& ok) {
    gas_prims<M>(q, p, pr, ok);
    pr[5] = M::sqrt_(M::div(p.gam * pr[2], q[0], ok), ok);
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ void roe(const R* pl, const R* pr, const P& p, R& uh, R& vh,
                                             R& c2, bool& ok) {
    constexpr int UN = NI - 1, UT = 2 - NI;
    R iws = M::rcp(pl[3] + pr[3], ok);
    uh = (pl[3] * pl[UN] + pr[3] * pr[UN]) * iws;
    vh = (pl[3] * pl[UT] + pr[3] * pr[UT]) * iws;
    R hh = (pl[4] + pr[4]) * iws;
    c2 = p.gm1 * (hh - (R)0.5 * (uh * uh + vh * vh));
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ void speeds(const R* pl, const R* pr, const P& p, R& s1,
                                                R& s2, R& c2, bool& ok) {
    constexpr int UN = NI - 1;
    R uh, vh;
    roe<NI, M>(pl, pr, p, uh, vh, c2, ok);
    R ch = M::sqrt_(c2, ok);
    s1 = nmin(pl[UN] - pl[5], uh - ch);
    s2 = nmax(pr[UN] + pr[5], uh + ch);
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ void solve(const R* ql, const R* qr, const R* pl, const R* pr,
                                               const R*, const R*, const P& p, R (&W)[NW][NEQ],
                                               R (&s)[NW], R (&am)[NEQ], R (&ap)[NEQ],
                                               bool& ok) {
    constexpr int TI = 3 - NI, UN = NI - 1;
    R s1, s2, c2;
    speeds<NI, M>(pl, pr, p, s1, s2, c2, ok);
    R ul = pl[UN], ur = pr[UN];
    R fl[NEQ], fr[NEQ];
    fl[0] = ql[NI]; fl[NI] = ql[NI] * ul + pl[2]; fl[TI] = ql[TI] * ul; fl[3] = ul * (ql[3] + pl[2]);
    fr[0] = qr[NI]; fr[NI] = qr[NI] * ur + pr[2]; fr[TI] = qr[TI] * ur; fr[3] = ur * (qr[3] + pr[2]);
    R inv = M::rcp(s1 - s2, ok);
    R n0 = nmin(s1, (R)0), n1 = nmin(s2, (R)0);
    R p0 = nmax(s1, (R)0), p1 = nmax(s2, (R)0);
#pragma unroll
    for (int m = 0; m < NEQ; ++m) {
      R df = fr[m] - fl[m];
      R dq = qr[m] - ql[m];
      W[0][m] = (df - s2 * dq) * inv;   // q_m - q_l
      W[1][m] = (s1 * dq - df) * inv;   // q_r - q_m
      am[m] = n0 * W[0][m] + n1 * W[1][m];
      ap[m] = p0 * W[0][m] + p1 * W[1][m];
    }
    s[0] = s1; s[1] = s2;
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ int probe(const R* ql, const R* qr, const R* pl, const R* pr,
                                              const R*, const R*, const P& p, R& smax, bool& ok) {
    int c = finite_code<R, NEQ>(ql, qr);
    if (c) { smax = (R)0; return c; }
    if (bad_pos(ql[0])) { smax = (R)0; return 3; }
    if (bad_pos(qr[0])) { smax = (R)0; return 4; }
    if (bad_pos(pl[2])) { smax = (R)0; return 5; }
    if (bad_pos(pr[2])) { smax = (R)0; return 6; }
    return probe_fast<NI, M>(ql, qr, pl, pr, (const R*)nullptr, (const R*)nullptr, p, smax, ok);
  }

  template <class R, class P>
  __device__ static __forceinline__ bool cell_ok(const R* q, const R*, const R* pr, const P&) {
    return all_finite<R, NEQ>(q) && !bad_pos(q[0]) && !bad_pos(pr[2]);
  }
  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ int probe_fast(const R*, const R*, const R* pl, const R* pr,
                                                   const R*, const R*, const P& p, R& smax,
                                                   bool& ok) {
    R s1, s2, c2;
    speeds<NI, M>(pl, pr, p, s1, s2, c2, ok);
    if (!(c2 > (R)0)) { smax = (R)0; return 7; }
    smax = nmax(fabs(s1), fabs(s2));
    return 0;
  }
};

// ---------------------------------------------------------------------------
// shallow water, Roe + Harten entropy fix (builder-owned; oracle rp_shallow_roe)
//   prims: {u = hu*(1/h), v = hv*(1/h), sqrt(h)}
struct ShallowRoe {
  static constexpr int NEQ = 3, NW = 3, NAUX = 0, NPR = 3;
  static constexpr bool STATIC_SPEEDS = false;
  static constexpr bool HAS_BOUND = true;   // bound_cell: CFL candidate filter
  // W2 = a2 (0, 0, 1): only the transverse slot
  template <int NI> __host__ __device__ static constexpr bool wzero(int w, int m) { return w == 1 && m != 3 - NI; }
  template <class R> struct Params { R grav, sqg; };

  template <class M, class R, class P>
  __device__ static __forceinline__ void prims(const R* q, const R*, const P&, R* pr, bool& ok) {
    R rh = M::rcp(q[0], ok);
    pr[0] = q[1] * rh;
    pr[1] = q[2] * rh;
    pr[2] = M::sqrt_(q[0], ok);
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ void roe(const R* ql, const R* qr, const R* pl, const R* pr,
                                             const P& p, R& uh, R& vh, R& ch, bool& ok) {
    constexpr int UN = NI - 1, UT = 2 - NI;
    R iws = M::rcp(pl[2] + pr[2], ok);
    uh = (pl[2] * pl[UN] + pr[2] * pr[UN]) * iws;
    vh = (pl[2] * pl[UT] + pr[2] * pr[UT]) * iws;
    ch = M::sqrt_(p.grav * ((R)0.5 * (ql[0] + qr[0])), ok);
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ void solve(const R* ql, const R* qr, const R* pl, const R* pr,
                                               const R*, const R*, const P& p, R (&W)[NW][NEQ],
                                               R (&s)[NW], R (&am)[NEQ], R (&ap)[NEQ],
                                               bool& ok) {
    constexpr int TI = 3 - NI, UN = NI - 1;
    R uh, vh, ch;
    roe<NI, M>(ql, qr, pl, pr, p, uh, vh, ch, ok);
    R d0 = qr[0] - ql[0];
    R d1 = qr[NI] - ql[NI];
    R d2 = qr[TI] - ql[TI];
    // 0.5/c == 0.5 * (1/c) bit for bit (power-of-two scaling commutes with
    // rounding), and the reciprocal is the cheaper sequence
    R i2c = (R)0.5 * M::rcp(ch, ok);
    R s1 = uh - ch, s3 = uh + ch;
    R a1 = (s3 * d0 - d1) * i2c;
    R a2 = d2 - vh * d0;
    R a3 = (d1 - s1 * d0) * i2c;
    W[0][0] = a1;   W[0][NI] = a1 * s1;  W[0][TI] = a1 * vh;
    W[1][0] = (R)0; W[1][NI] = (R)0;     W[1][TI] = a2;
    W[2][0] = a3;   W[2][NI] = a3 * s3;  W[2][TI] = a3 * vh;
    s[0] = s1; s[1] = uh; s[2] = s3;
    // Harten entropy fix on families 1 and 3 (LeVeque 2002 §15.3.5)
    R cl = p.sqg * pl[2], cr = p.sqg * pr[2];
    R ul = pl[UN], ur = pr[UN];
    R del1 = nmax((R)0, (ur - cr) - (ul - cl));
    R del3 = nmax((R)0, (ur + cr) - (ul + cl));
    R f1 = fabs(s1), f2 = fabs(uh), f3 = fabs(s3);
    if (f1 < del1) f1 = M::div(s1 * s1 + del1 * del1, (R)2 * del1, ok);
    if (f3 < del3) f3 = M::div(s3 * s3 + del3 * del3, (R)2 * del3, ok);
    R am1 = (R)0.5 * (s1 - f1), am2 = (R)0.5 * (uh - f2), am3 = (R)0.5 * (s3 - f3);
    R ap1 = (R)0.5 * (s1 + f1), ap2 = (R)0.5 * (uh + f2), ap3 = (R)0.5 * (s3 + f3);
    am[0] = am1 * W[0][0] + am3 * W[2][0];
    am[NI] = am1 * W[0][NI] + am3 * W[2][NI];
    am[TI] = am1 * W[0][TI] + am2 * a2 + am3 * W[2][TI];
    ap[0] = ap1 * W[0][0] + ap3 * W[2][0];
    ap[NI] = ap1 * W[0][NI] + ap3 * W[2][NI];
    ap[TI] = ap1 * W[0][TI] + ap2 * a2 + ap3 * W[2][TI];
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ int probe(const R* ql, const R* qr, const R* pl, const R* pr,
                                              const R*, const R*, const P& p, R& smax, bool& ok) {
    int c = finite_code<R, NEQ>(ql, qr);
    if (c) { smax = (R)0; return c; }
    if (bad_pos(ql[0])) { smax = (R)0; return 3; }
    if (bad_pos(qr[0])) { smax = (R)0; return 4; }
    return probe_fast<NI, M>(ql, qr, pl, pr, (const R*)nullptr, (const R*)nullptr, p, smax, ok);
  }

  template <class R, class P>
  __device__ static __forceinline__ bool cell_ok(const R* q, const R*, const R*, const P&) {
    return all_finite<R, NEQ>(q) && !bad_pos(q[0]);
  }
  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ int probe_fast(const R* ql, const R* qr, const R* pl,
                                                   const R* pr, const R*, const R*, const P& p,
                                                   R& smax, bool& ok) {
    R uh, vh, ch;
    roe<NI, M>(ql, qr, pl, pr, p, uh, vh, ch, ok);
    // |uh| never exceeds max(|uh-c|, |uh+c|) for c >= 0 (rounding is monotone)
    smax = nmax(fabs(uh - ch), fabs(uh + ch));
    return 0;
  }

  // CFL candidate filter (k_speeds_b).  probe_fast's max |s| is |uh| + ch up
  // to rounding, uh is a convex combination of u_l, u_r and ch = sqrt(g (h_l
  // + h_r) / 2) <= sqrt(g max(h_l, h_r)), so for the edge
  //     max|s| <= (max(bx_l, bx_r) + max(bc_l, bc_r)) * MARGIN
  // with bx = |hu| / h (by = |hv| / h) and bc = sqrt(g) sqrt(h) from the
  // approximate seeds.  Returns false (edge must be probed exactly) unless the
  // cell is admissible and every quantity is in the seeds' safe range.
  template <class R, class P>
  __device__ static __forceinline__ bool bound_cell(const R* q, const R*, const P& p, R& bx,
                                                    R& by, R& bc) {
    const R h = q[0];
    const R r = BoundMath::rcp(h);
    bx = fabs(q[1]) * r;
    by = fabs(q[2]) * r;
    bc = p.sqg * (h * BoundMath::rsqrt(h));
    return BoundMath::pos_ok(h) && BoundMath::abs_ok(q[1]) && BoundMath::abs_ok(q[2]) &&
           BoundMath::small(bx) && BoundMath::small(by) && BoundMath::small(bc);
  }

  // Tile form (k_update_w epilogue -> k_speeds_t): integer maxima of the
  // high words over the tile's new cells, a = {max |hu|, max |hv|, max h,
  // min h} (signed, so a negative, NaN or zero depth shows up at either end),
  // then, from the accumulators folded over the cells an edge set reads,
  // bx = max|hu| / min h >= every cell's |u|, by likewise, bc = sqrt(g)
  // sqrt(max h), and the edge-speed bounds bx + bc (x), by + bc (y); +inf
  // when any cell leaves the seeds' range.
  static constexpr bool HAS_TILE = true;
  static constexpr int NACC = 4;
  static constexpr unsigned ACC_MIN = 0x8u;   // slots reduced with min
  __device__ static __forceinline__ void acc_init(int (&a)[NACC]) {
    a[0] = 0; a[1] = 0; a[2] = INT_MIN; a[3] = INT_MAX;
  }
  template <class R, class P>
  __device__ static __forceinline__ void tile_acc(const R* q, const P&, int (&a)[NACC]) {
    const int h = BoundMath::hw(q[0]);
    a[0] = max(a[0], BoundMath::hw(q[1]) & 0x7fffffff);
    a[1] = max(a[1], BoundMath::hw(q[2]) & 0x7fffffff);
    a[2] = max(a[2], h);
    a[3] = min(a[3], h);
  }
  template <class R, class P>
  __device__ static __forceinline__ void tile_bound(const int (&a)[NACC], const P& p, R& bndx,
                                                    R& bndy) {
    const int lo = BoundMath::hw_lo<R>(), hi = BoundMath::hw_hi<R>();
    const R hmin = BoundMath::lb<R>(a[3]);
    const R bx = BoundMath::ub<R>(a[0]) / hmin;
    const R by = BoundMath::ub<R>(a[1]) / hmin;
    const R bc = p.sqg * sqrt(BoundMath::ub<R>(a[2]));
    const bool ok = a[0] < hi && a[1] < hi && a[2] < hi && a[3] >= lo &&
                    BoundMath::small(bx) && BoundMath::small(by) && BoundMath::small(bc);
    bndx = ok ? bx + bc : (R)INFINITY;
    bndy = ok ? by + bc : (R)INFINITY;
  }
};

// ---------------------------------------------------------------------------
// scalar advection with constant velocity (u, v) — reference kernels.py:163-178
//   one wave W = qr - ql at s = u (x) or v (y); amdq = min(s,0) W, apdq = max(s,0) W
//   with Python's min/max on floats: min(s, 0.0) = 0.0 if 0.0 < s else s
struct Advection {
  static constexpr int NEQ = 1, NW = 1, NAUX = 0, NPR = 0;
  static constexpr bool STATIC_SPEEDS = true;
  // Tile form for row-strip shards (k_speeds_t): the speeds are static, so a
  // tile only needs probing if one of its new cells is inadmissible (then
  // the checked probe finds the reference-order first interface); a[0] =
  // "some cell is not finite" over the tile.  Aux is static: the first
  // pre-pass after an upload probes every tile.
  static constexpr bool HAS_TILE = true;
  static constexpr int NACC = 4;
  static constexpr unsigned ACC_MIN = 0x0u;
  __device__ static __forceinline__ void acc_init(int (&a)[NACC]) {
    a[0] = 0; a[1] = 0; a[2] = 0; a[3] = 0;
  }
  template <class R, class P>
  __device__ static __forceinline__ void tile_acc(const R* q, const P&, int (&a)[NACC]) {
    a[0] = max(a[0], all_finite<R, NEQ>(q) ? 0 : 1);
  }
  template <class R, class P>
  __device__ static __forceinline__ void tile_bound(const int (&a)[NACC], const P&, R& bndx,
                                                    R& bndy) {
    bndx = bndy = a[0] ? (R)INFINITY : (R)0;
  }
  template <int NI> __host__ __device__ static constexpr bool wzero(int, int) { return false; }
  template <class R> struct Params { R u, v; };

  template <class M, class R, class P>
  __device__ static __forceinline__ void prims(const R*, const R*, const P&, R*, bool&) {}

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ void solve(const R* ql, const R* qr, const R*, const R*,
                                               const R*, const R*, const P& p, R (&W)[NW][NEQ],
                                               R (&s)[NW], R (&am)[NEQ], R (&ap)[NEQ], bool&) {
    const R sp = (NI == 1) ? p.u : p.v;
    const R jump = qr[0] - ql[0];
    const R mn = ((R)0 < sp) ? (R)0 : sp;
    const R mx = ((R)0 > sp) ? (R)0 : sp;
    W[0][0] = jump;
    s[0] = sp;
    am[0] = mn * jump;
    ap[0] = mx * jump;
  }

  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ int probe(const R* ql, const R* qr, const R*, const R*,
                                              const R*, const R*, const P& p, R& smax, bool&) {
    smax = fabs((NI == 1) ? p.u : p.v);
    return finite_code<R, NEQ>(ql, qr);
  }

  template <class R, class P>
  __device__ static __forceinline__ bool cell_ok(const R* q, const R*, const R*, const P&) {
    return all_finite<R, NEQ>(q);
  }
  template <int NI, class M, class R, class P>
  __device__ static __forceinline__ int probe_fast(const R*, const R*, const R*, const R*,
                                                   const R*, const R*, const P& p, R& smax,
                                                   bool&) {
    smax = fabs((NI == 1) ? p.u : p.v);
    return 0;
  }
};

// ---------------------------------------------------------------------------
// the fp32 throughput mode (WS_FP32_FAST): the same plugin, a distinct type
// so its kernels -- compiled in ws_inst_fast_*.cu with FMA contraction and
// approximate division / square root -- never share a symbol with the
// bitwise fp32 kernels
template <class S> struct Fast : S {};

// ---------------------------------------------------------------------------
// wave limiters (oracle phi(); LeVeque 2002 §6.9)
template <int LIM, class R> __device__ __forceinline__ R limiter_phi(R th) {
  if (LIM == LIM_MINMOD) return nmax((R)0, nmin((R)1, th));
  if (LIM == LIM_SUPERBEE) return nmax((R)0, nmax(nmin((R)1, (R)2 * th), nmin((R)2, th)));
  if (LIM == LIM_MC) return nmax((R)0, nmin(nmin((R)0.5 * ((R)1 + th), (R)2), (R)2 * th));
  return (R)1;
}

}  // namespace ws
