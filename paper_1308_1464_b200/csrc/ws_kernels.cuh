// ws_kernels.cuh — the step kernels.
//
//   k_speeds  : CFL pre-pass.  Every reference edge (x: i in [0,nx], j in
//               [0,ny); y: i in [0,nx), j in [0,ny], solve_x / solve_y, sweep.py:111-163, 250)
//               is probed: admissibility in the reference order and max |s|,
//               reduced warp-shuffle -> block -> one atomicMax per CTA.
//   k_update  : fused edge + update kernel.  One CTA owns a TX x TY tile; the
//               tile plus an H-cell halo is staged in shared memory once,
//               per-cell primitives are computed once per cell, every edge
//               is solved once per tile, waves are limited against their
//               upwind neighbour, and the donor-cell update (reference order,
//               apply_update cells -= ..., sweep.py:275-277) plus the correction flux are applied in
//               registers.  No fluctuation arrays ever reach HBM.  The last
//               CTA to finish commits the step (report, t, counters).
//   k_to_soa / k_to_aos / k_static_speed : layout conversion, acoustics setup.
#pragma once
#include <climits>
#include <type_traits>

#include "ws_solvers.cuh"

#ifndef WS_LB3
#define WS_LB3 1
#endif
#ifndef WS_LNW3
#define WS_LNW3 10   // warps per line-kernel CTA for 1-3 component systems
#endif
#ifndef WS_F32_MINB
#define WS_F32_MINB 4   // fp32 10-warp line-kernel CTAs per SM, 1-3 components (48 registers)
#endif
// Line-kernel variants chosen per solver and precision from A/B runs on one
// B200 (profiles/r2_s5_ab.md, profiles/r2_s6_ab.md); -1 = that policy, 0 / 1 force a form for
// experiments.  The update kernel sits at its register cap (64 at three
// CTAs per SM), where fewer instructions do not always mean a faster kernel.
#ifndef WS_ROWSTAGE
#define WS_ROWSTAGE -1  // halo tile staged a row per warp (uniform row addressing)
#endif
#ifndef WS_ROWSTORE
#define WS_ROWSTORE -1  // tile stored a row per warp
#endif
#ifndef WS_LIMSEL
#define WS_LIMSEL -1    // limiter ratio: one select on phi instead of guarded operands
#endif
#ifndef WS_STGB
#define WS_STGB -1      // staged cells per thread and batch of loads (0: all at once)
#endif
// L2 band prefetch (band_prefetch): the CTAs of a tile row share out the halo
// band of the tile row ~WS_PFD CTAs ahead -- about the number of co-resident
// CTAs (148 SMs x 3) -- one cp.async.bulk.prefetch.L2 per row segment, so the
// staging loads hit L2 instead of HBM
#ifndef WS_L2PF
#define WS_L2PF 1
#endif
#ifndef WS_PFD
#define WS_PFD 444
#endif
// Interior tiles staged by a non-inlined row-per-warp helper (stage_inner)
// on NWARP - 1 warps while the last warp evaluates the step control
#ifndef WS_FASTSTAGE
#define WS_FASTSTAGE -1
#endif
#ifndef WS_GAS2
#define WS_GAS2 1   // 4-component fp64 on 10-warp CTAs, two per SM (0: 15 warps, one, persistent)
#endif

namespace ws {

template <class S, class R> struct LinePolicy {
  static constexpr bool F64 = sizeof(R) == 8;
  // C4 +3.7 %, C3 +1.7 % (two-wave solvers); three-wave fp64 -4 %, fp32 -1.5 %
  static constexpr bool LIMSEL = WS_LIMSEL < 0 ? (F64 && S::NW == 2) : (WS_LIMSEL != 0);
  // C3 (two CTAs per SM, 96 registers) +1.3 % / +1.6 %, all three +3.1 %;
  // three-component fp64 at 64 registers: -10 % (C5), -2 % (C4)
  static constexpr bool ROWSTAGE = WS_ROWSTAGE < 0 ? (F64 && S::NEQ >= 4) : (WS_ROWSTAGE != 0);
  static constexpr bool ROWSTORE = WS_ROWSTORE < 0 ? (F64 && S::NEQ >= 4) : (WS_ROWSTORE != 0);
  // loads of one batch in flight per thread: (NEQ + NAUX) * batch values.
  // Five fp64 values per cell (C4) times four cells spill at 64 registers
  // (batches of 2: no spills, same speed); C3 +3.2 % on top of ROWSTAGE, fp32
  // +0.7 % (C5) / +1.6 % (C4); three-component fp64 (C5, C2) -1 %
  // interior tiles through stage_inner: C4 +2.2 %, fp32 +1.6 % (C4, C5); the
  // three-wave fp64 kernel loses its register allocation (C5 -2.7 %, C2 -2.7 %),
  // four-component fp64 (row staging already) +-0
  static constexpr bool FASTSTAGE =
      WS_FASTSTAGE < 0 ? (!F64 || (S::NW == 2 && S::NEQ <= 3)) : (WS_FASTSTAGE != 0);
  static constexpr int STGB = WS_STGB < 0 ? ((!F64 || S::NEQ >= 4 || S::NEQ + S::NAUX >= 5) ? 2 : 0)
                                          : WS_STGB;
};

// bytes [p, p + n) towards L2, no register or shared-memory destination
// (p 16-byte aligned, n a multiple of 16)
__device__ __forceinline__ void l2_prefetch_bulk(const void* p, unsigned n) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(n) : "memory");
}

// Band prefetch for the line kernel: the CTAs of one tile row share out the
// halo band (HW rows x components, first row jb) of a tile row further down
// -- about WS_PFD CTAs ahead, the co-resident count -- as whole row
// segments, one cp.async.bulk.prefetch.L2 each.  A hint: nothing waits for
// it.  Not inlined: the update kernel sits at its register cap and its
// allocation must not depend on this code.
template <class R, int NEQ, int NAUX, int HW>
__device__ __noinline__ void band_prefetch(const R* q, const R* aux, int nx, int ny,
                                           long long pitch, long long rstride, long long astride,
                                           int ntx, int txv, int jb) {
  constexpr int NC = NEQ + NAUX, NRC = HW * NC;
  const int nseg = ntx >= NRC ? ntx / NRC : 1;
  for (int it = txv; it < NRC * nseg; it += ntx) {
    const int sg = it / NRC, rc = it - sg * NRC;
    const int ly = rc / NC, c = rc - ly * NC;
    const int gj = jb + ly;
    if (gj < 0 || gj >= ny) continue;
    const int g0 = (int)((long long)nx * sg / nseg);
    const int g1 = (int)((long long)nx * (sg + 1) / nseg);
    const R* rowp = c < NEQ ? q + (long long)(gj + 2) * rstride + c * pitch
                            : aux + (long long)(gj + 2) * astride + (c - NEQ) * pitch;
    const unsigned long long lo = (unsigned long long)(rowp + g0) & ~15ull;
    const unsigned long long hi = (unsigned long long)(rowp + g1) & ~15ull;
    if (hi > lo) l2_prefetch_bulk((const void*)lo, (unsigned)(hi - lo));
  }
}

// --------------------------------------------------------------------------
// block reductions
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

template <int NT>
__device__ __forceinline__ unsigned long long block_max_u64(unsigned long long v,
                                                            unsigned long long* sbuf) {
  v = warp_max_u64(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sbuf[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = (lane < NT / 32) ? sbuf[lane] : 0ull;
    v = warp_max_u64(v);
  }
  return v;  // valid in thread 0
}

// limiter ratio (W_up . W) / (W . W), 0 for a zero wave (oracle correction_flux)
template <class R> __device__ __forceinline__ R theta(R dup, R dow) {
  if (dow == (R)0) return (R)0;
  bool ok = true;
  const R q = FastMath::div(dup, dow, ok);
  return ok ? q : dup / dow;
}

// per-cell primitives with FastMath; IEEE re-evaluation if a range test failed
template <class S, class R, class P>
__device__ __forceinline__ void prims_fast(const R* q, const R* a, const P& p, R* pr) {
  bool ok = true;
  S::template prims<FastMath>(q, a, p, pr, ok);
  if (!ok) {
    bool d = true;
    S::template prims<IeeeMath>(q, a, p, pr, d);
  }
}

// --------------------------------------------------------------------------
// CFL / admissibility pre-pass.  Tile of TX x TY "edge cells" (x-edge = left
// edge of the cell, y-edge = bottom edge, plus the domain's last column/row),
// NT threads, each TX*TY/NT cells.  Per-cell admissibility (finite, positive)
// is evaluated once per cell while staging; a tile whose cells all pass uses
// the check-free probe (only the pairwise Roe c^2 test remains).
template <class S, class R, int TX, int TY, int NT>
__global__ void __launch_bounds__(NT)
k_speeds(const R* __restrict__ q, const R* __restrict__ aux, const Layout L,
         const typename S::template Params<R> P, const int cur, DevState* __restrict__ ds) {
  constexpr int NEQ = S::NEQ, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int HX = TX + 1, HY = TY + 1, HC = HX * HY;
  constexpr int NA1 = NAUX > 0 ? NAUX : 1, NP1 = NPR > 0 ? NPR : 1;
  constexpr int KC = TX * TY / NT;
  static_assert(KC * NT == TX * TY, "tile must be a multiple of the block");
  __shared__ R sQ[NEQ][HC];
  __shared__ R sA[NA1][NAUX > 0 ? HC : 1];
  __shared__ R sP[NP1][NPR > 0 ? HC : 1];
  __shared__ unsigned long long sred[2][NT / 32];
  __shared__ int s_skip;
  const int tid = threadIdx.x;
  // one L2 read per CTA (the flags cannot change during this kernel: only the
  // update kernel's commit writes them); broadcast through shared memory
  if (tid == 0) s_skip = __ldcg(&ds->err) | __ldcg(&ds->finished);
  __syncthreads();
  if (s_skip) return;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  // tile cell (lx, ly) = cell (i0 - 1 + lx, j0 - 1 + ly)
  const bool inner = i0 >= 1 && i0 + TX <= L.nx && j0 >= 1 && j0 + TY <= L.ny;
  bool ok = true;
  for (int idx = tid; idx < HC; idx += NT) {
    const int lx = idx % HX, ly = idx / HX;
    int gi = i0 - 1 + lx, gj = j0 - 1 + ly;
    if (!inner) { gi = map_i(gi, L); gj = map_j(gj, L); }
    R qc[NEQ], ac[NA1], pc[NP1];
    const R* src = q + row_off(gj, L) + gi;
#pragma unroll
    for (int c = 0; c < NEQ; ++c) { qc[c] = src[c * L.pitch]; sQ[c][idx] = qc[c]; }
    if (NAUX > 0) {
      const R* asrc = aux + (long long)(gj + 2) * L.astride + gi;
#pragma unroll
      for (int c = 0; c < NAUX; ++c) { ac[c] = asrc[c * L.pitch]; sA[c][idx] = ac[c]; }
    }
    if (NPR > 0) {
      prims_fast<S>(qc, ac, P, pc);
#pragma unroll
      for (int c = 0; c < NPR; ++c) sP[c][idx] = pc[c];
    }
    ok = ok && S::cell_ok(qc, ac, pc, P);
  }
  const bool clean = __syncthreads_and(ok);

  R mx = (R)0, my = (R)0;
  unsigned long long key = ~0ull;
  auto edge = [&](auto ni_tag, int cl, int cr, int dir, int ei, int ej) {
    constexpr int NI = decltype(ni_tag)::value;
    R ql[NEQ], qr[NEQ], al[NA1], ar[NA1], pl[NP1], pr[NP1];
#pragma unroll
    for (int c = 0; c < NEQ; ++c) { ql[c] = sQ[c][cl]; qr[c] = sQ[c][cr]; }
#pragma unroll
    for (int c = 0; c < NAUX; ++c) { al[c] = sA[c][cl]; ar[c] = sA[c][cr]; }
#pragma unroll
    for (int c = 0; c < NPR; ++c) { pl[c] = sP[c][cl]; pr[c] = sP[c][cr]; }
    R sm;
    bool ok = true;
    int code;
    if (clean) {
      code = S::template probe_fast<NI, FastMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
      if (!ok) code = S::template probe_fast<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
    } else {
      code = S::template probe<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
    }
    if (code) {
      unsigned long long k = err_key(dir, ei, L.j_off + ej, (code & 0xff) - 1, code >> 8, L.nx);
      key = k < key ? k : key;
    }
    return sm;
  };
  using NX = std::integral_constant<int, 1>;
  using NY = std::integral_constant<int, 2>;
#pragma unroll
  for (int kc = 0; kc < KC; ++kc) {
    const int cidx = tid + kc * NT;
    const int li = cidx % TX, lj = cidx / TX;
    const int i = i0 + li, j = j0 + lj;
    if (i <= L.nx && j < L.ny) {
      R s = edge(NX{}, (lj + 1) * HX + li, (lj + 1) * HX + li + 1, 0, i, j);
      mx = nmax(mx, s);   // NaN-free unless inadmissible (flagged)
    }
    if (i < L.nx && j < L.ny_edges_y) {
      R s = edge(NY{}, lj * HX + li + 1, (lj + 1) * HX + li + 1, 1, i, j);
      my = nmax(my, s);
    }
  }
  if (key != ~0ull) atomicMax(&ds->slot[cur][2], NKEY_MAX - key);
  // both maxima in one warp-shuffle tree
  unsigned long long bx = Bits<R>::to(mx), by = Bits<R>::to(my);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long wx = __shfl_xor_sync(0xffffffffu, bx, o);
    unsigned long long wy = __shfl_xor_sync(0xffffffffu, by, o);
    bx = wx > bx ? wx : bx;
    by = wy > by ? wy : by;
  }
  const int lane = tid & 31, wid = tid >> 5;
  if (lane == 0) { sred[0][wid] = bx; sred[1][wid] = by; }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) {
      bx = sred[0][w] > bx ? sred[0][w] : bx;
      by = sred[1][w] > by ? sred[1][w] : by;
    }
    atomicMax(&ds->slot[cur][0], bx);
    atomicMax(&ds->slot[cur][1], by);
  }
}

// spin (acquire, system scope) until a device counter written by other
// shards reaches `need`; gives up with ERR_WAIT_TIMEOUT (never in a healthy run)
__device__ __forceinline__ void wait_counter(const unsigned long long* cnt, unsigned long long need,
                                             DevState* ds) {
  long long spins = 0;
  while (ld_acquire_sys(cnt) < need) {
    if (__ldcg(&ds->err)) return;
    __nanosleep(128);
    if (++spins > (1ll << 24)) { atomicCAS(&ds->err, 0, ERR_WAIT_TIMEOUT); return; }
  }
}

// --------------------------------------------------------------------------
// CFL / admissibility pre-pass, register form (the default).  One warp owns a
// strip of 31 edge columns x KC edge rows: lane l holds cell column
// x0 - 1 + l, so the x-edge left of its cell pairs it with lane l-1 (one
// shuffle per used field), and the warp marches up its rows keeping the
// previous row's cell in registers for the y-edge below.  No shared-memory
// staging, no per-cell index division; prims are evaluated (31+1)/31 x
// (KC+1)/KC times per cell.  Per edge, the check-free probe runs when both
// cells are admissible — exactly what the checked probe computes for them —
// and the checked probe (reference stage order) otherwise.
template <class S, class R, int KC, int NWS, int UNR, int MINB>
__global__ void __launch_bounds__(NWS * 32, MINB)
k_speeds_w(const R* __restrict__ q, const R* __restrict__ aux, const Layout L,
           const typename S::template Params<R> P, const int cur, const int part,
           DevState* __restrict__ ds) {
  constexpr int NEQ = S::NEQ, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int NA1 = NAUX > 0 ? NAUX : 1, NP1 = NPR > 0 ? NPR : 1;
  __shared__ unsigned long long sred[2][NWS];
  __shared__ int s_skip;
  // warp index via lane-0 broadcast = known warp-uniform (see k_update_w)
  const int tid = threadIdx.x, lane = tid & 31, wid = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const unsigned long long t_start = L.trace ? gtimer() : 0ull;
  // everything below reads the previous update's output; the next update may
  // launch only after that update completed, i.e. after this wait returned
  pdl_wait();
  if (L.hsides > 0 && part != 1) {
    // device-side halos: the neighbours' updates pushed this step's ghost
    // rows; wait for all of them (the update launched after us stages ghost
    // rows too, so the trigger comes after this wait)
    if (tid == 0) wait_counter(&ds->harrive, (unsigned long long)L.hsides * (unsigned long long)__ldcg(&ds->seq), ds);
    __syncthreads();
  }
  pdl_trigger();
  const int ci = blockIdx.x * 31 - 1 + lane;                 // this lane's cell column
  const int gi = map_i(ci < L.nx ? ci : L.nx, L);
  // part 2 runs two CTA rows: the first, and the one holding edge row ny
  const int brow = (part == 2 && blockIdx.y == 1) ? (L.ny_edges_y - 1) / (KC * NWS) : blockIdx.y;
  const int jb = (brow * NWS + wid) * KC;                      // first edge row of the warp
  // part (see Impl::speeds): the y-edges that read received ghost rows are
  // those of row 0 and, on a top shard whose high ghost rows come from a
  // (periodic) neighbour, of row ny; part 1 skips them, part 2 keeps only them
  const bool xcol = lane >= 1 && ci <= L.nx && part != 2;     // owns x-edge ci
  const bool ycol = lane >= 1 && ci < L.nx;                   // owns y-edge column ci
  const int ytop = (L.hi == ROWS_MEMORY && L.ny_edges_y > L.ny) ? L.ny : -1;

  // warps whose rows jb-1 .. jb+KC+1 are all interior skip the y mapping
  const bool inner_rows = jb >= 1 && jb + KC + 1 < L.ny;
  auto load = [&](int r, R (&qc)[NEQ], R (&ac)[NA1]) {
    const int gj = inner_rows ? r : map_j(r < L.ny ? r : L.ny, L);
    const R* src = q + row_off(gj, L) + gi;
#pragma unroll
    for (int c = 0; c < NEQ; ++c) qc[c] = src[c * L.pitch];
    if (NAUX > 0) {
      const R* asrc = aux + (long long)(gj + 2) * L.astride + gi;
#pragma unroll
      for (int c = 0; c < NAUX; ++c) ac[c] = asrc[c * L.pitch];
    }
  };
  // the first rows' loads go out before the run-flag barrier (they are
  // in-bounds whatever the flags say; a skipped step just drops them)
  R qp[NEQ], ap[NA1], qn[NEQ], an[NA1], qn2[NEQ], an2[NA1];
  load(jb - 1, qp, ap);
  load(jb, qn, an);
  load(jb + 1, qn2, an2);                   // two rows in flight ahead of the compute
  if (tid == 0) s_skip = __ldcg(&ds->err) | __ldcg(&ds->finished);
  __syncthreads();
  if (s_skip) return;
  auto cell = [&](const R (&qc)[NEQ], const R (&ac)[NA1], R (&pc)[NP1]) -> bool {
    if (NPR > 0) prims_fast<S>(qc, ac, P, pc);
    return S::cell_ok(qc, ac, pc, P);
  };

  R mx = (R)0, my = (R)0;
  unsigned long long key = ~0ull;
  auto probe = [&](auto ni_tag, const R* ql, const R* qr, const R* pl, const R* pr,
                   const R* al, const R* ar, bool clean, int dir, int ei, int ej) -> R {
    constexpr int NI = decltype(ni_tag)::value;
    R sm;
    bool ok = true;
    int code;
    if (clean) {
      code = S::template probe_fast<NI, FastMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
      if (!ok) code = S::template probe_fast<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
    } else {
      code = S::template probe<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
    }
    if (code) {
      unsigned long long k = err_key(dir, ei, L.j_off + ej, (code & 0xff) - 1, code >> 8, L.nx);
      key = k < key ? k : key;
    }
    return sm;
  };
  using NX = std::integral_constant<int, 1>;
  using NY = std::integral_constant<int, 2>;

  // edge rows this warp owns: [jb, jb + nk), nothing past the last edge row
  const int rows = L.ny > L.ny_edges_y ? L.ny : L.ny_edges_y;
  const int nk = rows - jb < KC ? rows - jb : KC;
  if (nk > 0) {
    R pp[NP1];
    bool okp = cell(qp, ap, pp);
#pragma unroll UNR
    for (int k = 0; k < KC; ++k) {
      if (k >= nk) break;
      const int r = jb + k;
      R qc[NEQ], ac[NA1], pc[NP1];
#pragma unroll
      for (int c = 0; c < NEQ; ++c) { qc[c] = qn[c]; qn[c] = qn2[c]; }
#pragma unroll
      for (int c = 0; c < NAUX; ++c) { ac[c] = an[c]; an[c] = an2[c]; }
      load(r + 2, qn2, an2);
      const bool okc = cell(qc, ac, pc);
      // left neighbour (lane - 1) of the current row
      R ql[NEQ], al[NA1], pl[NP1];
#pragma unroll
      for (int c = 0; c < NEQ; ++c) ql[c] = __shfl_up_sync(0xffffffffu, qc[c], 1);
#pragma unroll
      for (int c = 0; c < NAUX; ++c) al[c] = __shfl_up_sync(0xffffffffu, ac[c], 1);
#pragma unroll
      for (int c = 0; c < NPR; ++c) pl[c] = __shfl_up_sync(0xffffffffu, pc[c], 1);
      const bool okl = __shfl_up_sync(0xffffffffu, okc, 1);
      if (xcol && r < L.ny)
        mx = nmax(mx, probe(NX{}, ql, qc, pl, pc, al, ac, okl && okc, 0, ci, r));
      const bool ghost_edge = r == 0 || r == ytop;
      if (ycol && r < L.ny_edges_y && (part == 0 || (part == 2) == ghost_edge))
        my = nmax(my, probe(NY{}, qp, qc, pp, pc, ap, ac, okp && okc, 1, ci, r));
#pragma unroll
      for (int c = 0; c < NEQ; ++c) qp[c] = qc[c];
#pragma unroll
      for (int c = 0; c < NAUX; ++c) ap[c] = ac[c];
#pragma unroll
      for (int c = 0; c < NPR; ++c) pp[c] = pc[c];
      okp = okc;
    }
  }
  if (key != ~0ull) atomicMax(&ds->slot[cur][2], NKEY_MAX - key);
  unsigned long long bx = Bits<R>::to(mx), by = Bits<R>::to(my);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long wx = __shfl_xor_sync(0xffffffffu, bx, o);
    unsigned long long wy = __shfl_xor_sync(0xffffffffu, by, o);
    bx = wx > bx ? wx : bx;
    by = wy > by ? wy : by;
  }
  if (lane == 0) { sred[0][wid] = bx; sred[1][wid] = by; }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int w = 1; w < NWS; ++w) {
      bx = sred[0][w] > bx ? sred[0][w] : bx;
      by = sred[1][w] > by ? sred[1][w] : by;
    }
    atomicMax(&ds->slot[cur][0], bx);
    atomicMax(&ds->slot[cur][1], by);
    if (L.npeers > 0 && part != 1) {
      // device-side reduction across shards: the last CTA pushes this
      // shard's slot into every shard's slot (64-bit MAX, over NVLink for
      // peers) and then announces the push with a release increment
      __threadfence();
      if (atomicAdd(&ds->pdone, 1) == (int)(gridDim.x * gridDim.y) - 1) {
        __threadfence();
        ds->pdone = 0;
        const unsigned long long v0 = atomicOr(&ds->slot[cur][0], 0ull);
        const unsigned long long v1 = atomicOr(&ds->slot[cur][1], 0ull);
        const unsigned long long v2 = atomicOr(&ds->slot[cur][2], 0ull);
        for (int r = 0; r < L.npeers; ++r) {
          DevState* pr = L.peers[r];
          atomicMax_system(&pr->slot[cur][0], v0);
          atomicMax_system(&pr->slot[cur][1], v1);
          if (v2) atomicMax_system(&pr->slot[cur][2], v2);
        }
        __threadfence_system();
        for (int r = 0; r < L.npeers; ++r) atomicAdd_system(&L.peers[r]->arrive, 1ull);
      }
    }
    if (L.trace) trace_cta(L, 0, t_start);
  }
}

// cp.async (LDGSTS): global -> shared without a register round trip, so the
// next tile's loads are in flight while the current tile is computed
__device__ __forceinline__ void cp_async(void* smem, const double* g) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_async(void* smem, const float* g) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// --------------------------------------------------------------------------
// CFL / admissibility pre-pass with a candidate filter (solvers with
// S::HAS_BOUND; the default for them).  Same warp geometry as k_speeds_w, but
// an edge is probed exactly only if it can hold the step's maximum: every
// edge gets a cheap upper bound B_e >= max|s|_e from per-cell seeds
// (S::bound_cell, no IEEE division or square root), and with T any EXACT
// max|s| of some edge of the current state (a lower bound of the step's
// maximum M), an edge with B_e < T has max|s|_e <= B_e < T <= M and cannot
// change the maximum.  So
//     max over {e : B_e >= T} of max|s|_e  ==  M   (bit for bit),
// and edges whose cells are not provably admissible are always probed
// (checked probe: errors and their reference-order key are unchanged).
// T per warp: the exact max|s| at the edge where the previous step's maximum
// was found (DevState::hint, recorded by this kernel), the slot's running
// maximum of this step, and each lane's own running maximum.
template <class S, class = void> struct HasBound : std::false_type {};
template <class S> struct HasBound<S, std::enable_if_t<S::HAS_BOUND>> : std::true_type {};
// tile accumulators for the tile-filtered pre-pass (S::tile_acc / tile_bound)
template <class S, class = void> struct HasTile : std::false_type {};
template <class S> struct HasTile<S, std::enable_if_t<S::HAS_TILE>> : std::true_type {};
template <class S, class = void> struct NAcc { static constexpr int value = 4; };
template <class S> struct NAcc<S, std::enable_if_t<S::HAS_TILE>> {
  static constexpr int value = S::NACC;
};
template <class S, class = void> struct AccMin { static constexpr unsigned value = 0u; };
template <class S> struct AccMin<S, std::enable_if_t<S::HAS_TILE>> {
  static constexpr unsigned value = S::ACC_MIN;
};

constexpr unsigned long long HINT_IDX_MASK = (1ull << 29) - 1;
template <class R>
__device__ __forceinline__ unsigned long long hint_key(R s, long long idx) {
  const unsigned long long b = (unsigned long long)__double_as_longlong((double)s);
  const unsigned long long ix = (idx >= 0 && idx < (long long)HINT_IDX_MASK)
                                    ? (unsigned long long)idx : HINT_IDX_MASK;
  return ((b >> 29) << 29) | ix;
}

// Exact max|s| on the current state at the hint edge of direction dir (0: x,
// 1: y), or 0 when there is none, it is out of range, it reads ghost rows a
// split step has not received yet (part 1), or it is not admissible.
template <class S, class R>
__device__ __forceinline__ R hint_probe(const R* __restrict__ q, const R* __restrict__ aux,
                                        const Layout& L, const typename S::template Params<R>& P,
                                        const DevState* ds, int dir, int part, int ytop) {
  constexpr int NEQ = S::NEQ, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int NA1 = NAUX > 0 ? NAUX : 1, NP1 = NPR > 0 ? NPR : 1;
  const unsigned long long hk = __ldcg(&ds->hint[dir]);
  const long long idx = (long long)(hk & HINT_IDX_MASK);
  const long long w = dir == 0 ? (long long)L.nx + 1 : (long long)L.nx;
  const long long hj = idx / w;
  const int hi = (int)(idx - hj * w);
  const bool use = hk != 0ull && (dir == 0 ? hj < L.ny
                                           : (hj < L.ny_edges_y &&
                                              (part != 1 || (hj != 0 && hj != ytop))));
  if (!use) return (R)0;
  R ql[NEQ], qr[NEQ], al[NA1], ar[NA1], pl[NP1], pr[NP1];
  auto load_at = [&](int gcol, int gj, R (&qc)[NEQ], R (&ac)[NA1]) {
    const R* src = q + row_off(gj, L) + gcol;
#pragma unroll
    for (int c = 0; c < NEQ; ++c) qc[c] = __ldcg(src + c * L.pitch);
    if (NAUX > 0) {
      const R* asrc = aux + (long long)(gj + 2) * L.astride + gcol;
#pragma unroll
      for (int c = 0; c < NAUX; ++c) ac[c] = __ldcg(asrc + c * L.pitch);
    }
  };
  if (dir == 0) {
    load_at(map_i(hi - 1, L), (int)hj, ql, al);
    load_at(map_i(hi, L), (int)hj, qr, ar);
  } else {
    load_at(hi, map_j((int)hj - 1, L), ql, al);
    load_at(hi, map_j((int)hj < L.ny ? (int)hj : L.ny, L), qr, ar);
  }
  if (NPR > 0) { prims_fast<S>(ql, al, P, pl); prims_fast<S>(qr, ar, P, pr); }
  if (!(S::cell_ok(ql, al, pl, P) && S::cell_ok(qr, ar, pr, P))) return (R)0;
  bool ok = true;
  R sm;
  int code;
  if (dir == 0) {
    code = S::template probe_fast<1, FastMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
    if (!ok) code = S::template probe_fast<1, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
  } else {
    code = S::template probe_fast<2, FastMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
    if (!ok) code = S::template probe_fast<2, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
  }
  return code == 0 ? sm : (R)0;   // an inadmissible edge (Euler c^2 <= 0) gives no bound
}

template <class S, class R, int KC, int NWS, int MINB, int RING>
__global__ void __launch_bounds__(NWS * 32, MINB)
k_speeds_b(const R* __restrict__ q, const R* __restrict__ aux, const Layout L,
           const typename S::template Params<R> P, const int cur, const int part,
           DevState* __restrict__ ds) {
  constexpr int NEQ = S::NEQ, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int NA1 = NAUX > 0 ? NAUX : 1, NP1 = NPR > 0 ? NPR : 1;
  const R MARGIN = (R)BoundMath::MARGIN;
  __shared__ unsigned long long sred[2][NWS];
  __shared__ int s_skip;
  const int tid = threadIdx.x, lane = tid & 31, wid = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const unsigned long long t_start = L.trace ? gtimer() : 0ull;
  pdl_wait();
  if (L.hsides > 0 && part != 1) {
    if (tid == 0) wait_counter(&ds->harrive, (unsigned long long)L.hsides * (unsigned long long)__ldcg(&ds->seq), ds);
    __syncthreads();
  }
  pdl_trigger();
  const int ci = blockIdx.x * 31 - 1 + lane;
  const int gi = map_i(ci < L.nx ? ci : L.nx, L);
  const int brow = (part == 2 && blockIdx.y == 1) ? (L.ny_edges_y - 1) / (KC * NWS) : blockIdx.y;
  const int jb = (brow * NWS + wid) * KC;
  const bool xcol = lane >= 1 && ci <= L.nx && part != 2;
  const bool ycol = lane >= 1 && ci < L.nx;
  const int ytop = (L.hi == ROWS_MEMORY && L.ny_edges_y > L.ny) ? L.ny : -1;
  const bool inner_rows = jb >= 1 && jb + KC + 1 < L.ny;
  // per-thread ring of RING rows in shared memory, filled by cp.async: the
  // row loop keeps RING - 1 rows in flight without holding them in registers
  // (the pre-pass is bound by load latency once the per-edge work is gone).
  // Each lane reads back only the elements it copied itself: no warp sync.
  constexpr int NC = NEQ + NAUX;
  __shared__ R ring[RING][NC][NWS * 32];
  auto issue = [&](int t) {   // row jb - 1 + t into slot t % RING (always one group)
    if (t <= KC) {
      const int r = jb - 1 + t;
      const int gj = inner_rows ? r : map_j(r < L.ny ? r : L.ny, L);
      const R* src = q + row_off(gj, L) + gi;
#pragma unroll
      for (int c = 0; c < NEQ; ++c) cp_async(&ring[t % RING][c][tid], src + c * L.pitch);
      if (NAUX > 0) {
        const R* asrc = aux + (long long)(gj + 2) * L.astride + gi;
#pragma unroll
        for (int c = 0; c < NAUX; ++c) cp_async(&ring[t % RING][NEQ + c][tid], asrc + c * L.pitch);
      }
    }
    cp_commit();
  };
  auto take = [&](int t, R (&qc)[NEQ], R (&ac)[NA1]) {   // row jb - 1 + t, after its wait
#pragma unroll
    for (int c = 0; c < NEQ; ++c) qc[c] = ring[t % RING][c][tid];
#pragma unroll
    for (int c = 0; c < NAUX; ++c) ac[c] = ring[t % RING][NEQ + c][tid];
  };
#pragma unroll
  for (int t = 0; t < RING; ++t) issue(t);

  // the hint edges: lane 0 probes the x-edge, lane 1 the y-edge (exactly, on
  // the current state; a hint that reads rows still in flight is skipped)
  using NX = std::integral_constant<int, 1>;
  using NY = std::integral_constant<int, 2>;
  R gh = (R)0;
  if (lane < 2) gh = hint_probe<S>(q, aux, L, P, ds, lane, part, ytop);
  if (tid == 0) s_skip = __ldcg(&ds->err) | __ldcg(&ds->finished);
  __syncthreads();
  if (s_skip) { cp_wait<0>(); return; }
  // lower bounds: the hint edges and this step's running maxima (exact |s| of
  // current-state edges; in a sharded step possibly of other shards' edges)
  R tx = __shfl_sync(0xffffffffu, gh, 0), ty = __shfl_sync(0xffffffffu, gh, 1);
  tx = nmax(tx, Bits<R>::from(__ldcg(&ds->slot[cur][0])));
  ty = nmax(ty, Bits<R>::from(__ldcg(&ds->slot[cur][1])));

  R mx = (R)0, my = (R)0;
  unsigned long long key = ~0ull, kx = 0ull, ky = 0ull;
  auto probe = [&](auto ni_tag, const R* ql, const R* qr, const R* pl, const R* pr,
                   const R* al, const R* ar, bool clean, int dir, int ei, int ej) -> R {
    constexpr int NI = decltype(ni_tag)::value;
    R sm;
    bool ok = true;
    int code;
    if (clean) {
      code = S::template probe_fast<NI, FastMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
      if (!ok) code = S::template probe_fast<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
    } else {
      code = S::template probe<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
    }
    if (code) {
      unsigned long long k = err_key(dir, ei, L.j_off + ej, (code & 0xff) - 1, code >> 8, L.nx);
      key = k < key ? k : key;
    }
    return sm;
  };

  const int rows = L.ny > L.ny_edges_y ? L.ny : L.ny_edges_y;
  const int nk = rows - jb < KC ? rows - jb : KC;
  R qp[NEQ], ap[NA1];
  if (nk > 0) {
    cp_wait<RING - 1>();
    take(0, qp, ap);
    issue(RING);
    R byp, bcp, bxd;
    bool vp = S::bound_cell(qp, ap, P, bxd, byp, bcp);
#pragma unroll 1
    for (int k = 0; k < KC; ++k) {
      if (k >= nk) break;
      const int r = jb + k;
      R qc[NEQ], ac[NA1];
      cp_wait<RING - 1>();
      take(k + 1, qc, ac);
      issue(k + 1 + RING);
      R bxc, byc, bcc;
      const bool vc = S::bound_cell(qc, ac, P, bxc, byc, bcc);
      const R bxl = __shfl_up_sync(0xffffffffu, bxc, 1);
      const R bcl = __shfl_up_sync(0xffffffffu, bcc, 1);
      const bool vl = __shfl_up_sync(0xffffffffu, vc, 1);
      const R bndx = (nmax(bxl, bxc) + nmax(bcl, bcc)) * MARGIN;
      const R bndy = (nmax(byp, byc) + nmax(bcp, bcc)) * MARGIN;
      const bool candx = xcol && r < L.ny && (!(vl && vc) || !(bndx < nmax(tx, mx)));
      const bool ghost_edge = r == 0 || r == ytop;
      const bool candy = ycol && r < L.ny_edges_y && (part == 0 || (part == 2) == ghost_edge) &&
                         (!(vp && vc) || !(bndy < nmax(ty, my)));
      if (__any_sync(0xffffffffu, candx || candy)) {
        R pc[NP1];
        if (NPR > 0) prims_fast<S>(qc, ac, P, pc);
        const bool okc = S::cell_ok(qc, ac, pc, P);
        if (__any_sync(0xffffffffu, candx)) {
          R ql[NEQ], al[NA1], pl[NP1];
#pragma unroll
          for (int c = 0; c < NEQ; ++c) ql[c] = __shfl_up_sync(0xffffffffu, qc[c], 1);
#pragma unroll
          for (int c = 0; c < NAUX; ++c) al[c] = __shfl_up_sync(0xffffffffu, ac[c], 1);
#pragma unroll
          for (int c = 0; c < NPR; ++c) pl[c] = __shfl_up_sync(0xffffffffu, pc[c], 1);
          const bool okl = __shfl_up_sync(0xffffffffu, okc, 1);
          if (candx) {
            const R s = probe(NX{}, ql, qc, pl, pc, al, ac, okl && okc, 0, ci, r);
            mx = nmax(mx, s);
            const unsigned long long hk = hint_key(s, (long long)r * (L.nx + 1) + ci);
            kx = hk > kx ? hk : kx;
          }
        }
        if (candy) {
          R pp[NP1];
          if (NPR > 0) prims_fast<S>(qp, ap, P, pp);
          const bool okp = S::cell_ok(qp, ap, pp, P);
          const R s = probe(NY{}, qp, qc, pp, pc, ap, ac, okp && okc, 1, ci, r);
          my = nmax(my, s);
          const unsigned long long hk = hint_key(s, (long long)r * L.nx + ci);
          ky = hk > ky ? hk : ky;
        }
      }
#pragma unroll
      for (int c = 0; c < NEQ; ++c) qp[c] = qc[c];
#pragma unroll
      for (int c = 0; c < NAUX; ++c) ap[c] = ac[c];
      byp = byc; bcp = bcc; vp = vc;
    }
  }
  cp_wait<0>();
  if (key != ~0ull) atomicMax(&ds->slot[cur][2], NKEY_MAX - key);
  // the maxima and the hint keys: warp-shuffle trees, then one atomic per
  // CTA and value (hint keys only where some lane probed)
  unsigned long long bx = Bits<R>::to(mx), by = Bits<R>::to(my);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long wx = __shfl_xor_sync(0xffffffffu, bx, o);
    unsigned long long wy = __shfl_xor_sync(0xffffffffu, by, o);
    unsigned long long hx = __shfl_xor_sync(0xffffffffu, kx, o);
    unsigned long long hy = __shfl_xor_sync(0xffffffffu, ky, o);
    bx = wx > bx ? wx : bx;
    by = wy > by ? wy : by;
    kx = hx > kx ? hx : kx;
    ky = hy > ky ? hy : ky;
  }
  if (lane == 0) {
    if (kx) atomicMax(&ds->hint_acc[cur][0], kx);
    if (ky) atomicMax(&ds->hint_acc[cur][1], ky);
    sred[0][wid] = bx; sred[1][wid] = by;
  }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int w = 1; w < NWS; ++w) {
      bx = sred[0][w] > bx ? sred[0][w] : bx;
      by = sred[1][w] > by ? sred[1][w] : by;
    }
    if (bx) atomicMax(&ds->slot[cur][0], bx);
    if (by) atomicMax(&ds->slot[cur][1], by);
    if (L.npeers > 0 && part != 1) {
      __threadfence();
      if (atomicAdd(&ds->pdone, 1) == (int)(gridDim.x * gridDim.y) - 1) {
        __threadfence();
        ds->pdone = 0;
        const unsigned long long v0 = atomicOr(&ds->slot[cur][0], 0ull);
        const unsigned long long v1 = atomicOr(&ds->slot[cur][1], 0ull);
        const unsigned long long v2 = atomicOr(&ds->slot[cur][2], 0ull);
        for (int r = 0; r < L.npeers; ++r) {
          DevState* pr = L.peers[r];
          atomicMax_system(&pr->slot[cur][0], v0);
          atomicMax_system(&pr->slot[cur][1], v1);
          if (v2) atomicMax_system(&pr->slot[cur][2], v2);
        }
        __threadfence_system();
        for (int r = 0; r < L.npeers; ++r) atomicAdd_system(&L.peers[r]->arrive, 1ull);
      }
    }
    if (L.trace) trace_cta(L, 0, t_start);
  }
}

// --------------------------------------------------------------------------
// CFL / admissibility pre-pass over whole tiles (solvers with S::HAS_TILE:
// shallow water, Euler Roe / HLLE; the default for them).
//
// The update kernel that wrote the state also stored, per 29x29 tile, integer
// maxima / minima of its new cells (S::tile_acc) and probed one x- and one
// y-edge of the new state exactly (DevState::tnext: the edges where this
// step's maxima were found).  The x-edges a tile owns read cells of the tile
// and of its left neighbour (periodic: also the wrapped right one for the
// domain's last edge column), its y-edges the tile and the one below, so
// S::tile_bound over those accumulators gives B_x(tile) >= max|s| of each
// x-edge it owns (B_y likewise).  With T an exact max|s| of some edge of this state (tnext, the
// running slot maximum), a tile with B_x * MARGIN < T cannot hold the x
// maximum: its x-edges are not even loaded.  The others are probed exactly,
// so the step's maxima are bit-identical to probing every edge.  A cell that
// is inadmissible or outside the bound's range makes B infinite: its edges
// are always probed with the checked probe (errors and their reference-order
// key).  Without valid tile data (first step after an upload, another update
// path) every tile is a candidate.
//
// One kernel: CTA c decides tiles c, c + G, c + 2G, ... (G = grid size, so a
// cluster of candidate tiles spreads over many CTAs, i.e. SMs), one thread per
// tile, into a shared-memory list; then its warps probe the listed tiles'
// edge rows, one row per item.
constexpr int TILE_NG = 30;   // edge rows of a tile (29, +1 for the top boundary row)
constexpr int TILE_LIST = 2048;

template <class S, class R>
__device__ __forceinline__ void tile_decide(const int4* __restrict__ tm, int t, int ntx, int nty,
                                            const Layout& L, const typename S::template Params<R>& P,
                                            R tlx, R tly, bool& cx, bool& cy) {
  constexpr int NA = NAcc<S>::value, NV = NA / 4;
  constexpr unsigned MINS = AccMin<S>::value;
  const R MARGIN = (R)BoundMath::MARGIN;
  const int tx = t % ntx, ty = t / ntx;
  // x-edges of a tile read its own cells and the left tile's last column
  // (periodic: tile ntx-1 left of tile 0, tile 0 right of the last tile);
  // y-edges likewise with the tile below / above
  const bool px = L.bcx == BC_PERIODIC, py = L.bcy == BC_PERIODIC;
  auto fold = [&](int (&a)[NA], int x, int y) {
    const int4* e = tm + ((long long)y * ntx + x) * NV;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int4 w = __ldcg(e + k);
      const int v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int m = 0; m < 4; ++m)
        a[4 * k + m] = ((MINS >> (4 * k + m)) & 1u) ? min(a[4 * k + m], v[m]) : max(a[4 * k + m], v[m]);
    }
  };
  int ax[NA], ay[NA];
  S::acc_init(ax);
  fold(ax, tx, ty);
#pragma unroll
  for (int k = 0; k < NA; ++k) ay[k] = ax[k];
  if (tx > 0 || px) fold(ax, tx > 0 ? tx - 1 : ntx - 1, ty);
  if (px && tx == ntx - 1) fold(ax, 0, ty);
  if (ty > 0 || py) fold(ay, tx, ty > 0 ? ty - 1 : nty - 1);
  if (py && ty == nty - 1) fold(ay, tx, 0);
  R bx, by, dx_, dy_;
  S::tile_bound(ax, P, bx, dy_);
  S::tile_bound(ay, P, dx_, by);
  cx = !(bx * MARGIN < tlx);
  cy = !(by * MARGIN < tly);
}

template <class S, class R, int NWT>
__global__ void __launch_bounds__(NWT * 32, (S::NEQ >= 4 ? 2 : 4))
k_speeds_t(const R* __restrict__ q, const R* __restrict__ aux, const int4* __restrict__ tmax,
           const Layout L, const typename S::template Params<R> P, const int cur, const int SPL,
           DevState* __restrict__ ds) {
  constexpr int NEQ = S::NEQ, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int NA1 = NAUX > 0 ? NAUX : 1, NP1 = NPR > 0 ? NPR : 1;
  constexpr int LW = 29, NT = NWT * 32;
  __shared__ unsigned s_list[TILE_LIST];
  __shared__ int s_cnt, s_ok;
  __shared__ R s_t[2];
  const int tid = threadIdx.x, lane = tid & 31, wid = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const unsigned long long t_start = L.trace ? gtimer() : 0ull;
  pdl_wait();
  if (L.hsides > 0) {
    // device-side halos: the neighbours' updates pushed this step's ghost
    // rows; wait for them (the update launched after us stages ghost rows
    // too, so the trigger comes after this wait)
    if (tid == 0) wait_counter(&ds->harrive, (unsigned long long)L.hsides * (unsigned long long)__ldcg(&ds->seq), ds);
    __syncthreads();
  }
  pdl_trigger();
  const int ntx = (L.nx + LW - 1) / LW, nty = (L.ny + LW - 1) / LW, nt = ntx * nty;
  if (tid == 0) {
    const int fl = __ldcg(&ds->err) | __ldcg(&ds->finished);
    const int ok = __ldcg(&ds->tmax_ok[cur]);
    R t0, t1;
    if constexpr (S::STATIC_SPEEDS) {
      // a static-speed shard: its maxima are the upload's (the slot carries
      // them to the reduction); only tiles holding a bad cell are probed
      const unsigned long long b0 = __ldcg(&ds->static_bits[0]), b1 = __ldcg(&ds->static_bits[1]);
      if (blockIdx.x == 0 && !fl) { atomicMax(&ds->slot[cur][0], b0); atomicMax(&ds->slot[cur][1], b1); }
      t0 = Bits<R>::from(b0); t1 = Bits<R>::from(b1);
    } else {
      t0 = nmax(Bits<R>::from(__ldcg(&ds->tnext[cur][0])), Bits<R>::from(__ldcg(&ds->slot[cur][0])));
      t1 = nmax(Bits<R>::from(__ldcg(&ds->tnext[cur][1])), Bits<R>::from(__ldcg(&ds->slot[cur][1])));
    }
    s_ok = fl ? -1 : ok;
    s_t[0] = t0; s_t[1] = t1;
    s_cnt = 0;
  }
  __syncthreads();
  const bool skip = s_ok < 0;
  if (!skip) {
    const int4* tm = tmax + (long long)cur * nt * (NAcc<S>::value / 4);
    const R tlx = s_t[0], tly = s_t[1];
    // virtual index v = tile * SPL + part: the SPL parts of a tile (rows
    // part, part + SPL, ...) land on SPL consecutive CTAs, which decide it
    // redundantly and probe its rows in parallel
    const long long nv = (long long)nt * SPL;
    for (long long v = blockIdx.x + (long long)tid * gridDim.x; v < nv; v += (long long)NT * gridDim.x) {
      const int t = (int)(v / SPL), part = (int)(v - (long long)t * SPL);
      bool cx = true, cy = true;
      if (s_ok) tile_decide<S, R>(tm, t, ntx, nty, L, P, tlx, tly, cx, cy);
      // a shard's y-edges next to ghost rows in memory read a neighbour's
      // cells, which no tile maxima here describe: always probed
      const int ty = t / ntx;
      if ((L.lo == ROWS_MEMORY && ty == 0) || (L.hi == ROWS_MEMORY && ty == nty - 1)) cy = true;
      if (cx || cy) {
        // entry: tile (28 bits) | part (2 bits, SPL <= 4) | cx << 30 | cy << 31
        const int slot = atomicAdd(&s_cnt, 1);
        if (slot < TILE_LIST)
          s_list[slot] = (unsigned)t | ((unsigned)part << 28) | (cx ? 1u << 30 : 0u) |
                         (cy ? 1u << 31 : 0u);
      }
    }
  }
  __syncthreads();
  // the host sizes the grid so a CTA lists at most NT * SPL <= TILE_LIST
  // tiles (ws_host.cuh); should that ever break, the step fails loudly
  // instead of overrunning shared memory
  if (s_cnt > TILE_LIST) {
    if (tid == 0) { atomicCAS(&ds->err, 0, ERR_INTERNAL); WS_CHK(L, false, CHK_TILE_LIST); }
    return;
  }
  // an item is a run of TR consecutive edge rows of a listed tile; part s of
  // a tile takes the runs s, s + SPL, ...
  constexpr int TR = S::NEQ >= 4 ? 4 : 1;       // gas prims are dear: march runs
  constexpr int NRUN = (TILE_NG + TR - 1) / TR;
  const int ngs = (NRUN + SPL - 1) / SPL;       // runs of one part
  const int nitems = skip ? 0 : s_cnt * ngs;

  R mx = (R)0, my = (R)0;
  unsigned long long key = ~0ull, kx = 0ull, ky = 0ull;
  auto probe = [&](auto ni_tag, const R* ql, const R* qr, const R* pl, const R* pr,
                   const R* al, const R* ar, bool clean, int dir, int ei, int ej) -> R {
    constexpr int NI = decltype(ni_tag)::value;
    R sm;
    bool ok = true;
    int code;
    if (clean) {
      code = S::template probe_fast<NI, FastMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
      if (!ok) code = S::template probe_fast<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
    } else {
      code = S::template probe<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, ok);
    }
    if (code) {
      unsigned long long k = err_key(dir, ei, L.j_off + ej, (code & 0xff) - 1, code >> 8, L.nx);
      key = k < key ? k : key;
    }
    return sm;
  };
  using NX = std::integral_constant<int, 1>;
  using NY = std::integral_constant<int, 2>;

  for (int item = wid; item < nitems; item += NWT) {
    const unsigned ent = s_list[item / ngs];
    const int tile = (int)(ent & ((1u << 28) - 1u));
    const int run = (int)((ent >> 28) & 3u) + SPL * (item % ngs);
    const bool cx = (ent >> 30) & 1u, cy = (ent >> 31) & 1u;
    const int i0 = (tile % ntx) * LW, j0 = (tile / ntx) * LW;
    // edges owned: x-edges ei in [i0, iend) on rows [j0, min(j0+29, ny));
    // y-edges ci in [i0, min(i0+29, nx)) on rows [j0, rend)
    const int iend = i0 + LW >= L.nx ? L.nx + 1 : i0 + LW;
    const int rend = j0 + LW >= L.ny ? L.ny_edges_y : j0 + LW;
    const int g0 = run * TR;
    const int rb = j0 + g0;
    int nr = rend - rb;
    nr = nr < TR ? nr : TR;
    if (g0 + nr > TILE_NG) nr = TILE_NG - g0;
    if (run >= NRUN || nr <= 0) continue;
    const int ci = i0 - 1 + lane;
    const int gi = map_i(ci < L.nx ? ci : L.nx, L);
    const bool xc = cx && lane >= 1 && ci < iend;
    const bool yc = cy && lane >= 1 && ci < (i0 + LW < L.nx ? i0 + LW : L.nx);
    // all TR + 1 rows of the run in flight at once
    R qb[TR + 1][NEQ], ab[TR + 1][NA1];
#pragma unroll
    for (int k = 0; k <= TR; ++k) {
      if (k <= nr) {
        const int rr = rb - 1 + k;
        const int gj = map_j(rr < L.ny ? rr : L.ny, L);
        WS_CHK(L, row_readable(gj, L) && gi >= 0 && gi < L.nx, CHK_PREPASS_READ);
        const R* src = q + row_off(gj, L) + gi;
#pragma unroll
        for (int c = 0; c < NEQ; ++c) qb[k][c] = __ldcg(src + c * L.pitch);
        if (NAUX > 0) {
          const R* asrc = aux + (long long)(gj + 2) * L.astride + gi;
#pragma unroll
          for (int c = 0; c < NAUX; ++c) ab[k][c] = __ldcg(asrc + c * L.pitch);
        }
      }
    }
    R pp[NP1];
    bool okp = true;
    if (cy) {   // the row below the run: its prims only feed y-edges
      if (NPR > 0) prims_fast<S>(qb[0], ab[0], P, pp);
      okp = S::cell_ok(qb[0], ab[0], pp, P);
    }
#pragma unroll
    for (int k = 1; k <= TR; ++k) {
      if (k > nr) break;
      const int r = rb - 1 + k;
      R pc[NP1];
      if (NPR > 0) prims_fast<S>(qb[k], ab[k], P, pc);
      const bool okc = S::cell_ok(qb[k], ab[k], pc, P);
      if (cx) {
        R ql[NEQ], al[NA1], pl[NP1];
#pragma unroll
        for (int c = 0; c < NEQ; ++c) ql[c] = __shfl_up_sync(0xffffffffu, qb[k][c], 1);
#pragma unroll
        for (int c = 0; c < NAUX; ++c) al[c] = __shfl_up_sync(0xffffffffu, ab[k][c], 1);
#pragma unroll
        for (int c = 0; c < NPR; ++c) pl[c] = __shfl_up_sync(0xffffffffu, pc[c], 1);
        const bool okl = __shfl_up_sync(0xffffffffu, okc, 1);
        if (xc && r < L.ny) {
          const R sv = probe(NX{}, ql, qb[k], pl, pc, al, ab[k], okl && okc, 0, ci, r);
          mx = nmax(mx, sv);
          const unsigned long long hk = hint_key(sv, (long long)r * (L.nx + 1) + ci);
          kx = hk > kx ? hk : kx;
        }
      }
      if (yc && r < L.ny_edges_y) {
        const R sv = probe(NY{}, qb[k - 1], qb[k], pp, pc, ab[k - 1], ab[k], okp && okc, 1, ci, r);
        my = nmax(my, sv);
        const unsigned long long hk = hint_key(sv, (long long)r * L.nx + ci);
        ky = hk > ky ? hk : ky;
      }
#pragma unroll
      for (int c = 0; c < NPR; ++c) pp[c] = pc[c];
      okp = okc;
    }
  }
  // per-warp results: at most one atomic per value and warp
  if (nitems > 0) {
  if (key != ~0ull) atomicMax(&ds->slot[cur][2], NKEY_MAX - key);
  unsigned long long bxs = Bits<R>::to(mx), bys = Bits<R>::to(my);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long wx = __shfl_xor_sync(0xffffffffu, bxs, o);
    unsigned long long wy = __shfl_xor_sync(0xffffffffu, bys, o);
    unsigned long long hx = __shfl_xor_sync(0xffffffffu, kx, o);
    unsigned long long hy = __shfl_xor_sync(0xffffffffu, ky, o);
    bxs = wx > bxs ? wx : bxs;
    bys = wy > bys ? wy : bys;
    kx = hx > kx ? hx : kx;
    ky = hy > ky ? hy : ky;
  }
  if (lane == 0) {
    if (bxs) atomicMax(&ds->slot[cur][0], bxs);
    if (bys) atomicMax(&ds->slot[cur][1], bys);
    if (kx) atomicMax(&ds->hint_acc[cur][0], kx);
    if (ky) atomicMax(&ds->hint_acc[cur][1], ky);
  }
  }
  if (L.npeers > 0) {
    // device-side reduction across shards: the last CTA pushes this shard's
    // slot into every shard's slot (64-bit MAX, over NVLink for peers) and
    // announces the push with a release increment (as k_speeds_w)
    __threadfence();
    __syncthreads();
    if (tid == 0 && atomicAdd(&ds->pdone, 1) == (int)gridDim.x - 1) {
      __threadfence();
      ds->pdone = 0;
      const unsigned long long v0 = atomicOr(&ds->slot[cur][0], 0ull);
      const unsigned long long v1 = atomicOr(&ds->slot[cur][1], 0ull);
      const unsigned long long v2 = atomicOr(&ds->slot[cur][2], 0ull);
      for (int r = 0; r < L.npeers; ++r) {
        DevState* pr = L.peers[r];
        atomicMax_system(&pr->slot[cur][0], v0);
        atomicMax_system(&pr->slot[cur][1], v1);
        if (v2) atomicMax_system(&pr->slot[cur][2], v2);
      }
      __threadfence_system();
      for (int r = 0; r < L.npeers; ++r) atomicAdd_system(&L.peers[r]->arrive, 1ull);
    }
  }
  if (L.trace && tid == 0) trace_cta(L, 0, t_start);
}

// --------------------------------------------------------------------------
// commit: run by thread 0 of the last CTA of an update kernel
template <class R>
__device__ __forceinline__ void commit_step(DevState* ds, const StepArgs& A, const Ctl& c,
                                            const Layout& L) {
  volatile DevState* v = ds;
  unsigned long long nkey = atomicOr(&ds->slot[A.cur][2], 0ull);
  if (v->err == 0) {
    if (c.finished) {
      v->finished = 1;
    } else if (nkey != 0ull) {
      v->err = ERR_KERNEL; v->err_key = NKEY_MAX - nkey; v->err_step = v->steps;
    } else if (c.stationary) {
      v->err = ERR_STATIONARY; v->err_step = v->steps;
    } else {
      long long n = v->nrep;
      Report r;
      r.dt = c.dt;
      r.cfl = c.dt * (c.msx / A.dx + c.msy / A.dy);   // cfl, driver.py:221
      r.msx = c.msx; r.msy = c.msy;
      ds->rep[n % REPCAP] = r;
      v->nrep = n + 1;
      v->steps = v->steps + 1;
      v->t = v->t + c.dt;
    }
  }
  // tile maxima of the state this step wrote: valid only after a committed
  // step of an update that stored them (k_speeds_t probes every tile otherwise)
  v->tmax_ok[A.cur ^ 1] = (A.tmax != nullptr && v->err == 0 && !c.finished && !c.stationary) ? 1 : 0;
  // the filter hint of the next pre-pass: where this step's maxima were found
  // (kept when this step's pre-pass recorded none, e.g. the exact pre-pass)
  if (v->hint_acc[A.cur][0]) v->hint[0] = v->hint_acc[A.cur][0];
  if (v->hint_acc[A.cur][1]) v->hint[1] = v->hint_acc[A.cur][1];
  v->hint_acc[A.cur][0] = 0ull; v->hint_acc[A.cur][1] = 0ull;
  // this step's slot is consumed; it is the accumulator of the step after next
  v->slot[A.cur][0] = 0ull; v->slot[A.cur][1] = 0ull; v->slot[A.cur][2] = 0ull;
  // a skipped step (t_final reached, error, stationary: the same decision on
  // every shard) stored no rows, but still releases the neighbours once, so
  // their halo-arrival counts stay hsides x seq
  if (c.skip) {
    __threadfence_system();
    if (L.nds_lo) atomicAdd_system(&L.nds_lo->harrive, 1ull);
    if (L.nds_hi) atomicAdd_system(&L.nds_hi->harrive, 1ull);
  }
  v->seq = v->seq + 1;
  __threadfence();
  v->done = 0;
}

// --------------------------------------------------------------------------
// fused edge + update kernel
template <class S, int ORDER, int TX, int TY>
struct TileGeom {
  static constexpr int NEQ = S::NEQ, NW = S::NW, NAUX = S::NAUX, NPR = S::NPR;
  static constexpr int H = (ORDER == 2) ? 2 : 1;
  static constexpr int HX = TX + 2 * H, HY = TY + 2 * H, HC = HX * HY;
  static constexpr int NEXC = TX + 2 * H - 1;   // x-edges per tile row
  static constexpr int NEX = NEXC * TY;
  static constexpr int NEYR = TY + 2 * H - 1;   // y-edge rows
  static constexpr int NEY = TX * NEYR;
  static constexpr int NEST = NEX > NEY ? NEX : NEY;
  static constexpr int NIX = (TX + 1) * TY, NIY = TX * (TY + 1);
  static constexpr int NIST = NIX > NIY ? NIX : NIY;
  static constexpr int NWS = NW * NEQ + NW;       // wave record (waves + speeds)
  static constexpr int NFL = (ORDER == 2 ? 3 : 2) * NEQ;  // amdq, apdq [, F~]
  static constexpr int EBUF = (ORDER == 2) ? (NEST * NWS > NIST * NFL ? NEST * NWS : NIST * NFL)
                                           : NIST * NFL;
  // double-buffered q and aux tiles + primitives + edge records
  template <class R> static constexpr size_t smem_bytes() {
    return sizeof(R) * (size_t)((2 * NEQ + 2 * NAUX + NPR) * HC + EBUF);
  }
};

// --------------------------------------------------------------------------
// FUSED CFL epilogue: max |s| and admissibility of the NEXT step's state,
// computed while q_new is still in shared memory.  Every reference edge is
// probed exactly once: edges inside a tile by that tile; extrapolated
// domain-boundary edges (ghost == boundary cell) by the boundary tile; an
// edge on a border shared by two tiles (or the periodic wrap) by whichever
// of the two finishes SECOND — it sees the other's q_new through a per-border
// counter (+1 per side per step; odd previous value = the other side is
// done), so nothing ever waits.  Single-shard only (shard borders need the
// exchanged halo, the multi-shard path keeps the k_speeds pre-pass).
template <class S, class R, int TX, int TY, int NT, int H>
__device__ __forceinline__ void next_step_speeds(
    R* sQ, const R* sA, R* sP, const R* __restrict__ qn, const R* __restrict__ aux,
    const Layout& L, const typename S::template Params<R>& P, const StepArgs& A, int i0, int j0,
    int tc, int tr, int ntx, int nty, int* s_second, R& nmx, R& nmy, unsigned long long& nkey) {
  constexpr int NEQ = S::NEQ, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int HX = TX + 2 * H, HC = HX * (TY + 2 * H);
  constexpr int NA1 = NAUX > 0 ? NAUX : 1, NP1 = NPR > 0 ? NPR : 1;
  static_assert(2 * TX + 2 * TY <= NT, "one thread per border edge");
  const int tid = threadIdx.x;
  const int nxv = min(TX, L.nx - i0), nyv = min(TY, L.ny - j0);
  const bool perx = L.bcx == BC_PERIODIC, pery = L.bcy == BC_PERIODIC;
  __syncthreads();   // q_new of the whole tile is in sQ

  // primitives of the tile's new cells
  for (int c2 = tid; c2 < TX * TY; c2 += NT) {
    const int idx = (c2 / TX + H) * HX + c2 % TX + H;
    R qc[NEQ], ac[NA1], pc[NP1];
#pragma unroll
    for (int c = 0; c < NEQ; ++c) qc[c] = sQ[c * HC + idx];
#pragma unroll
    for (int c = 0; c < NAUX; ++c) ac[c] = sA[c * HC + idx];
    prims_fast<S>(qc, ac, P, pc);
#pragma unroll
    for (int c = 0; c < NPR; ++c) sP[c * HC + idx] = pc[c];
  }
  __syncthreads();

  auto probe_smem = [&](auto ni_tag, int cl, int cr, int dir, int gi, int gj, R& mx) {
    constexpr int NI = decltype(ni_tag)::value;
    R ql[NEQ], qr[NEQ], al[NA1], ar[NA1], pl[NP1], pr[NP1];
#pragma unroll
    for (int c = 0; c < NEQ; ++c) { ql[c] = sQ[c * HC + cl]; qr[c] = sQ[c * HC + cr]; }
#pragma unroll
    for (int c = 0; c < NAUX; ++c) { al[c] = sA[c * HC + cl]; ar[c] = sA[c * HC + cr]; }
#pragma unroll
    for (int c = 0; c < NPR; ++c) { pl[c] = sP[c * HC + cl]; pr[c] = sP[c * HC + cr]; }
    R sm;
    bool okm = true;
    int code = S::template probe<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, okm);
    if (code) {
      unsigned long long k = err_key(dir, gi, L.j_off + gj, (code & 0xff) - 1, code >> 8, L.nx);
      nkey = k < nkey ? k : nkey;
    } else {
      mx = nmax(mx, sm);
    }
  };
  using NX = std::integral_constant<int, 1>;
  using NY = std::integral_constant<int, 2>;
  auto cidx = [&](int li, int lr) { return (lr + H) * HX + li + H; };

  // x-edges owned by the tile itself
  for (int e = tid; e < (TX + 1) * TY; e += NT) {
    const int le = e % (TX + 1), lr = e / (TX + 1);
    if (lr >= nyv || le > nxv) continue;
    const int gi = i0 + le;
    if (le > 0 && le < nxv) probe_smem(NX{}, cidx(le - 1, lr), cidx(le, lr), 0, gi, j0 + lr, nmx);
    else if (!perx && gi == 0) probe_smem(NX{}, cidx(0, lr), cidx(0, lr), 0, 0, j0 + lr, nmx);
    else if (!perx && gi == L.nx)
      probe_smem(NX{}, cidx(nxv - 1, lr), cidx(nxv - 1, lr), 0, gi, j0 + lr, nmx);
  }
  // y-edges owned by the tile itself
  for (int e = tid; e < TX * (TY + 1); e += NT) {
    const int li = e % TX, le = e / TX;
    if (li >= nxv || le > nyv) continue;
    const int gj = j0 + le;
    if (le > 0 && le < nyv) probe_smem(NY{}, cidx(li, le - 1), cidx(li, le), 1, i0 + li, gj, nmy);
    else if (!pery && gj == 0) probe_smem(NY{}, cidx(li, 0), cidx(li, 0), 1, i0 + li, 0, nmy);
    else if (!pery && gj == L.ny)
      probe_smem(NY{}, cidx(li, nyv - 1), cidx(li, nyv - 1), 1, i0 + li, gj, nmy);
  }

  // shared borders: left/right = vertical border ids, bottom/top = horizontal
  __syncthreads();
  if (tid == 0) {
    int* vb = A.borders;                 // [nty][ntx]: left border of tile column c
    int* hb = A.borders + ntx * nty;     // [nty][ntx]: bottom border of tile row r
    int s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    if (tc > 0 || perx) s0 = atomicAdd(&vb[tr * ntx + tc], 1) & 1;
    if (tc + 1 < ntx) s1 = atomicAdd(&vb[tr * ntx + tc + 1], 1) & 1;
    else if (perx) s1 = atomicAdd(&vb[tr * ntx + 0], 1) & 1;
    if (tr > 0 || pery) s2 = atomicAdd(&hb[tr * ntx + tc], 1) & 1;
    if (tr + 1 < nty) s3 = atomicAdd(&hb[(tr + 1) * ntx + tc], 1) & 1;
    else if (pery) s3 = atomicAdd(&hb[0 * ntx + tc], 1) & 1;
    __threadfence();
    s_second[0] = s0; s_second[1] = s1; s_second[2] = s2; s_second[3] = s3;
  }
  __syncthreads();

  auto probe_glob = [&](auto ni_tag, int il, int jl, int ir, int jr, int dir, int gi, int gj,
                        R& mx) {
    constexpr int NI = decltype(ni_tag)::value;
    R ql[NEQ], qr[NEQ], al[NA1], ar[NA1], pl[NP1], pr[NP1];
    const R* a = qn + row_off(jl, L) + il;
    const R* b = qn + row_off(jr, L) + ir;
#pragma unroll
    for (int c = 0; c < NEQ; ++c) { ql[c] = __ldcg(a + c * L.pitch); qr[c] = __ldcg(b + c * L.pitch); }
    if (NAUX > 0) {
      const R* xa = aux + (long long)(jl + 2) * L.astride + il;
      const R* xb = aux + (long long)(jr + 2) * L.astride + ir;
#pragma unroll
      for (int c = 0; c < NAUX; ++c) { al[c] = xa[c * L.pitch]; ar[c] = xb[c * L.pitch]; }
    }
    prims_fast<S>(ql, al, P, pl);
    prims_fast<S>(qr, ar, P, pr);
    R sm;
    bool okm = true;
    int code = S::template probe<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, okm);
    if (code) {
      unsigned long long k = err_key(dir, gi, L.j_off + gj, (code & 0xff) - 1, code >> 8, L.nx);
      nkey = k < nkey ? k : nkey;
    } else {
      mx = nmax(mx, sm);
    }
  };
  // left border: x-edge i0 (tile column > 0) or the periodic wrap pair (nx-1 | 0), edge 0
  if (s_second[0] && tid < nyv) {
    const int j = j0 + tid;
    if (tc > 0) probe_glob(NX{}, i0 - 1, j, i0, j, 0, i0, j, nmx);
    else probe_glob(NX{}, L.nx - 1, j, 0, j, 0, 0, j, nmx);
  }
  // right border
  if (s_second[1] && tid >= TY && tid < TY + nyv) {
    const int j = j0 + tid - TY;
    if (tc + 1 < ntx) probe_glob(NX{}, i0 + TX - 1, j, i0 + TX, j, 0, i0 + TX, j, nmx);
    else probe_glob(NX{}, L.nx - 1, j, 0, j, 0, 0, j, nmx);
  }
  // bottom border: y-edge j0 or the periodic wrap pair (ny-1 | 0), edge 0
  if (s_second[2] && tid >= 2 * TY && tid < 2 * TY + nxv) {
    const int i = i0 + tid - 2 * TY;
    if (tr > 0) probe_glob(NY{}, i, j0 - 1, i, j0, 1, i, j0, nmy);
    else probe_glob(NY{}, i, L.ny - 1, i, 0, 1, i, 0, nmy);
  }
  // top border
  if (s_second[3] && tid >= 2 * TY + TX && tid < 2 * TY + TX + nxv) {
    const int i = i0 + tid - 2 * TY - TX;
    if (tr + 1 < nty) probe_glob(NY{}, i, j0 + TY - 1, i, j0 + TY, 1, i, j0 + TY, nmy);
    else probe_glob(NY{}, i, L.ny - 1, i, 0, 1, i, 0, nmy);
  }
}


// Persistent CTAs walk the tiles (t = blockIdx.x, += gridDim.x).  Per tile:
// wait for its staged q(+aux) (issued one tile earlier), compute per-cell
// primitives, x sweep (solve -> limit -> records), x term, y sweep, y term +
// correction fluxes, store.  The next tile's loads overlap all of that.
template <class S, class R, int ORDER, int LIM, int TX, int TY, int NT, bool CHECKS, bool FUSED>
__global__ void __launch_bounds__(NT, (512 / NT > 0 ? 512 / NT : 1))
k_update(const R* __restrict__ q, const R* __restrict__ aux, R* __restrict__ qn, const Layout L,
         const typename S::template Params<R> P, const StepArgs A, DevState* __restrict__ ds) {
  using G = TileGeom<S, ORDER, TX, TY>;
  constexpr int NEQ = S::NEQ, NW = S::NW, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int H = G::H, HX = G::HX, HC = G::HC;
  constexpr int NEXC = G::NEXC, NEX = G::NEX, NEY = G::NEY, NEST = G::NEST, NIST = G::NIST;
  constexpr int KEX = (NEX + NT - 1) / NT, KEY = (NEY + NT - 1) / NT;
  constexpr int NCELL = TX * TY;
  constexpr int KC = (NCELL + NT - 1) / NT;
  constexpr int NA1 = NAUX > 0 ? NAUX : 1, NP1 = NPR > 0 ? NPR : 1;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sQb[2];
  R* sAb[2];
  sQb[0] = reinterpret_cast<R*>(smem_raw);
  sQb[1] = sQb[0] + NEQ * HC;
  sAb[0] = sQb[1] + NEQ * HC;
  sAb[1] = sAb[0] + NAUX * HC;
  R* sP = sAb[1] + NAUX * HC;
  R* sE = sP + NPR * HC;   // wave records (order 2), then fluctuation/flux records

  const int tid = threadIdx.x;
  const Ctl ctl = step_control<R>(A, ds, !CHECKS);   // identical in every thread
  const int ntx = (L.nx + TX - 1) / TX;
  const int nty = (L.ny + TY - 1) / TY;
  const int ntiles = ntx * nty;
  __shared__ unsigned long long s_red[NT / 32];
  __shared__ int s_second[4];
  R nmx = (R)0, nmy = (R)0;            // next step's max |s| (FUSED epilogue)
  unsigned long long nkey = ~0ull;     // next step's first inadmissible edge

  if (!ctl.skip) {
    const R dtdx = (R)(ctl.dt / A.dx);
    const R dtdy = (R)(ctl.dt / A.dy);
    unsigned long long key = ~0ull;

    auto stage = [&](int t, R* dq, R* da) {
      const int i0 = (t % ntx) * TX, j0 = (t / ntx) * TY;
      for (int idx = tid; idx < HC; idx += NT) {
        const int lx = idx % HX, ly = idx / HX;
        const int gi = map_i(i0 - H + lx, L), gj = map_j(j0 - H + ly, L);
        const R* src = q + row_off(gj, L) + gi;
#pragma unroll
        for (int c = 0; c < NEQ; ++c) cp_async(&dq[c * HC + idx], src + c * L.pitch);
        if (NAUX > 0) {
          const R* asrc = aux + (long long)(gj + 2) * L.astride + gi;
#pragma unroll
          for (int c = 0; c < NAUX; ++c) cp_async(&da[c * HC + idx], asrc + c * L.pitch);
        }
      }
      cp_commit();
    };

    int buf = 0;
    if ((int)blockIdx.x < ntiles) stage(blockIdx.x, sQb[0], sAb[0]);
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, buf ^= 1) {
      R* sQ = sQb[buf];
      R* sA = sAb[buf];
      const int i0 = (t % ntx) * TX, j0 = (t / ntx) * TY;
      const int tn = t + gridDim.x;
      if (tn < ntiles) { stage(tn, sQb[buf ^ 1], sAb[buf ^ 1]); cp_wait<1>(); }
      else cp_wait<0>();
      __syncthreads();

      // ---- per-cell primitives, once per staged cell
      if (NPR > 0) {
        for (int idx = tid; idx < HC; idx += NT) {
          R qc[NEQ], ac[NA1], pc[NP1];
#pragma unroll
          for (int c = 0; c < NEQ; ++c) qc[c] = sQ[c * HC + idx];
#pragma unroll
          for (int c = 0; c < NAUX; ++c) ac[c] = sA[c * HC + idx];
          prims_fast<S>(qc, ac, P, pc);
#pragma unroll
          for (int c = 0; c < NPR; ++c) sP[c * HC + idx] = pc[c];
        }
        __syncthreads();
      }

      R q1[KC][NEQ];

      // one sweep direction: solve -> (limit) -> fluctuation/flux records in sE
      auto sweep = [&](auto ni_tag) {
        constexpr int NI = decltype(ni_tag)::value;
        constexpr int NE = (NI == 1) ? NEX : NEY;
        constexpr int KE = (NI == 1) ? KEX : KEY;
        R fm[KE][NEQ], fp[KE][NEQ], ff[KE][NEQ];
#pragma unroll
        for (int k = 0; k < KE; ++k) {
          const int e = tid + k * NT;
          if (e < NE) {
            int cl, cr, ei, ej;
            if (NI == 1) {
              const int r = e / NEXC, c = e - r * NEXC;
              cl = (r + H) * HX + c; cr = cl + 1;
              ei = i0 - (H - 1) + c; ej = j0 + r;
            } else {
              const int r = e / TX, c = e - r * TX;
              cl = r * HX + c + H; cr = cl + HX;
              ei = i0 + c; ej = j0 - (H - 1) + r;
            }
            R ql[NEQ], qr[NEQ], al[NA1], ar[NA1], pl[NP1], pr[NP1];
#pragma unroll
            for (int c = 0; c < NEQ; ++c) { ql[c] = sQ[c * HC + cl]; qr[c] = sQ[c * HC + cr]; }
#pragma unroll
            for (int c = 0; c < NAUX; ++c) { al[c] = sA[c * HC + cl]; ar[c] = sA[c * HC + cr]; }
#pragma unroll
            for (int c = 0; c < NPR; ++c) { pl[c] = sP[c * HC + cl]; pr[c] = sP[c * HC + cr]; }
            R W[NW][NEQ], s[NW];
            bool oks = true;
            S::template solve<NI, FastMath>(ql, qr, pl, pr, al, ar, P, W, s, fm[k], fp[k], oks);
            if (!oks) S::template solve<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, W, s, fm[k], fp[k], oks);
            if (ORDER == 2) {
#pragma unroll
              for (int w = 0; w < NW; ++w) {
#pragma unroll
                for (int m = 0; m < NEQ; ++m) sE[(w * NEQ + m) * NEST + e] = W[w][m];
                sE[(NW * NEQ + w) * NEST + e] = s[w];
              }
            }
            if (CHECKS) {
              bool ref = (NI == 1) ? (ei >= 0 && ei <= L.nx && ej < L.ny)
                                   : (ei < L.nx && ej >= 0 && ej < L.ny_edges_y);
              if (ref) {
                R sm;
                bool okm = true;
                int code = S::template probe<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, okm);
                if (code) {
                  unsigned long long kk = err_key(NI - 1, ei, L.j_off + ej, (code & 0xff) - 1,
                                                  code >> 8, L.nx);
                  key = kk < key ? kk : key;
                }
              }
            }
          }
        }
        if (ORDER == 2) {
          __syncthreads();
          // limiter + correction flux on the inner edges
          const R dtdn = (NI == 1) ? dtdx : dtdy;
#pragma unroll
          for (int k = 0; k < KE; ++k) {
            const int e = tid + k * NT;
            bool inner = false;
            if (e < NE) {
              if (NI == 1) { const int c = e % NEXC; inner = (c >= H - 1) && (c <= TX + H - 1); }
              else { const int r = e / TX; inner = (r >= H - 1) && (r <= TY + H - 1); }
            }
            if (inner) {
              constexpr int STEP = (NI == 1) ? 1 : TX;
              R f[NEQ];
#pragma unroll
              for (int w = 0; w < NW; ++w) {
                R so = sE[(NW * NEQ + w) * NEST + e];
                const int up = (so > (R)0) ? e - STEP : e + STEP;
                R own[NEQ];
#pragma unroll
                for (int m = 0; m < NEQ; ++m) own[m] = sE[(w * NEQ + m) * NEST + e];
                R dup = sE[(w * NEQ) * NEST + up] * own[0];
                R dow = own[0] * own[0];
#pragma unroll
                for (int m = 1; m < NEQ; ++m) {
                  dup = dup + sE[(w * NEQ + m) * NEST + up] * own[m];
                  dow = dow + own[m] * own[m];
                }
                R th = theta(dup, dow);
                R ph = limiter_phi<LIM>(th);
                R a = fabs(so);
                R coef = a * ((R)1 - dtdn * a);
                R cph = coef * ph;
#pragma unroll
                for (int m = 0; m < NEQ; ++m) {
                  R wl = cph * own[m];
                  f[m] = (w == 0) ? wl : f[m] + wl;
                }
              }
#pragma unroll
              for (int m = 0; m < NEQ; ++m) ff[k][m] = (R)0.5 * f[m];
            }
          }
        }
        __syncthreads();
        // compact fluctuation (+ flux) records of the inner edges
#pragma unroll
        for (int k = 0; k < KE; ++k) {
          const int e = tid + k * NT;
          if (e < NE) {
            int ii = -1;
            if (NI == 1) {
              const int r = e / NEXC, c = e - r * NEXC;
              if (c >= H - 1 && c <= TX + H - 1) ii = r * (TX + 1) + (c - (H - 1));
            } else {
              const int r = e / TX, c = e - r * TX;
              if (r >= H - 1 && r <= TY + H - 1) ii = (r - (H - 1)) * TX + c;
            }
            if (ii >= 0) {
#pragma unroll
              for (int m = 0; m < NEQ; ++m) {
                sE[m * NIST + ii] = fm[k][m];
                sE[(NEQ + m) * NIST + ii] = fp[k][m];
                if (ORDER == 2) sE[(2 * NEQ + m) * NIST + ii] = ff[k][m];
              }
            }
          }
        }
        __syncthreads();
      };

      using NX = std::integral_constant<int, 1>;
      using NY = std::integral_constant<int, 2>;

      // ---- x sweep, then the reference's x term  q1 = q - dtdx*(apdq[i] + amdq[i+1])
      sweep(NX{});
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        const int cidx = tid + kc * NT;
        if (cidx < NCELL) {
          const int li = cidx % TX, lr = cidx / TX;
          const int el = lr * (TX + 1) + li, er = el + 1;
#pragma unroll
          for (int m = 0; m < NEQ; ++m) {
            R qc = sQ[m * HC + (lr + H) * HX + li + H];
            q1[kc][m] = qc - dtdx * (sE[(NEQ + m) * NIST + el] + sE[m * NIST + er]);
            if (ORDER == 2)
              q1[kc][m] = q1[kc][m] - dtdx * (sE[(2 * NEQ + m) * NIST + er] -
                                              sE[(2 * NEQ + m) * NIST + el]);
          }
        }
      }
      __syncthreads();

      // ---- y sweep, the y term, then the correction fluxes
      sweep(NY{});
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        const int cidx = tid + kc * NT;
        if (cidx < NCELL) {
          const int li = cidx % TX, lr = cidx / TX;
          const int el = lr * TX + li, eu = el + TX;
          const int gi = i0 + li, gj = j0 + lr;
          R out[NEQ];
#pragma unroll
          for (int m = 0; m < NEQ; ++m) {
            R v = q1[kc][m] - dtdy * (sE[(NEQ + m) * NIST + el] + sE[m * NIST + eu]);
            if (ORDER == 2)
              v = v - dtdy * (sE[(2 * NEQ + m) * NIST + eu] - sE[(2 * NEQ + m) * NIST + el]);
            out[m] = v;
          }
          if (gi < L.nx && gj < L.ny) {
            R* dst = qn + row_off(gj, L) + gi;
#pragma unroll
            for (int m = 0; m < NEQ; ++m) dst[m * L.pitch] = out[m];
          }
          if (FUSED) {
#pragma unroll
            for (int m = 0; m < NEQ; ++m) sQ[m * HC + (lr + H) * HX + li + H] = out[m];
          }
        }
      }
      if (FUSED) {
        __threadfence();   // q_new visible device-wide before the border counters
        next_step_speeds<S, R, TX, TY, NT, H>(sQ, sA, sP, qn, aux, L, P, A, i0, j0, t % ntx,
                                           t / ntx, ntx, nty, s_second, nmx, nmy, nkey);
      }
      __syncthreads();   // sQ/sP/sE of this tile are reused two tiles later
    }
    if (CHECKS && key != ~0ull) atomicMax(&ds->slot[A.cur][2], NKEY_MAX - key);
  }

  if (FUSED) {
    // the next step's CFL maxima / first error go to the other slot
    if (nkey != ~0ull) atomicMax(&ds->slot[A.cur ^ 1][2], NKEY_MAX - nkey);
    unsigned long long bx = block_max_u64<NT>(Bits<R>::to(nmx), s_red);
    __syncthreads();
    unsigned long long by = block_max_u64<NT>(Bits<R>::to(nmy), s_red);
    if (tid == 0) {
      atomicMax(&ds->slot[A.cur ^ 1][0], bx);
      atomicMax(&ds->slot[A.cur ^ 1][1], by);
    }
  }

  // ---- last CTA commits the step
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const int nblk = gridDim.x * gridDim.y;
    const int prev = atomicAdd(&ds->done, 1);
    if (prev == nblk - 1) {
      __threadfence();
      commit_step<R>(ds, A, ctl, L);
    }
  }
}

// FUSED epilogue helper: admissibility + max |s| of one edge of the NEXT
// state (cell-local tests already known through `clean`)
template <class S, class R, int NI>
__device__ __forceinline__ void probe_next(const R* ql, const R* qr, const R* pl, const R* pr,
                                           bool clean, const typename S::template Params<R>& P,
                                           const Layout& L, int gi, int gj, R& mx,
                                           unsigned long long& key) {
  R sm;
  bool ok = true;
  int code;
  if (clean) {
    code = S::template probe_fast<NI, FastMath>(ql, qr, pl, pr, (const R*)nullptr,
                                                (const R*)nullptr, P, sm, ok);
    if (!ok) code = S::template probe_fast<NI, IeeeMath>(ql, qr, pl, pr, (const R*)nullptr,
                                                         (const R*)nullptr, P, sm, ok);
  } else {
    code = S::template probe<NI, IeeeMath>(ql, qr, pl, pr, (const R*)nullptr, (const R*)nullptr,
                                           P, sm, ok);
  }
  if (code) {
    unsigned long long k = err_key(NI - 1, gi, L.j_off + gj, (code & 0xff) - 1, code >> 8, L.nx);
    key = k < key ? k : key;
  } else {
    mx = nmax(mx, sm);
  }
}

// Edges on the borders between LW x LW tiles (and the periodic wrap, reported
// as edge 0), probed on the new state after the FUSED update kernel: the
// only reference edges its epilogue cannot see.  One thread per edge.
template <class S, class R, int LW, int NT>
__global__ void __launch_bounds__(NT)
k_border(const R* __restrict__ q, const Layout L, const typename S::template Params<R> P,
         const int slot, DevState* __restrict__ ds) {
  constexpr int NEQ = S::NEQ, NPR = S::NPR, NP1 = NPR > 0 ? NPR : 1;
  __shared__ unsigned long long sred[2][NT / 32];
  __shared__ int s_skip;
  const int tid = threadIdx.x;
  if (tid == 0) s_skip = __ldcg(&ds->err) | __ldcg(&ds->finished);
  __syncthreads();
  if (s_skip) return;
  const int ntx = (L.nx + LW - 1) / LW, nty = (L.ny + LW - 1) / LW;
  const bool perx = L.bcx == BC_PERIODIC, pery = L.bcy == BC_PERIODIC;
  const int nvb = ntx - 1 + (perx ? 1 : 0), nhb = nty - 1 + (pery ? 1 : 0);
  const long long nv = (long long)nvb * L.ny, n = nv + (long long)nhb * L.nx;
  R mx = (R)0, my = (R)0;
  unsigned long long key = ~0ull;
  for (long long t = blockIdx.x * (long long)NT + tid; t < n; t += (long long)gridDim.x * NT) {
    int il, jl, ir, jr, gi, gj, dir;
    if (t < nv) {
      const int b = (int)(t / L.ny), j = (int)(t % L.ny);
      dir = 0; gj = j; jl = jr = j;
      if (b < ntx - 1) { gi = (b + 1) * LW; il = gi - 1; ir = gi; }
      else { gi = 0; il = L.nx - 1; ir = 0; }
    } else {
      const long long u = t - nv;
      const int b = (int)(u / L.nx), i = (int)(u % L.nx);
      dir = 1; gi = i; il = ir = i;
      if (b < nty - 1) { gj = (b + 1) * LW; jl = gj - 1; jr = gj; }
      else { gj = 0; jl = L.ny - 1; jr = 0; }
    }
    R ql[NEQ], qr[NEQ], pl[NP1], pr[NP1];
    const R* a = q + row_off(jl, L) + il;
    const R* b = q + row_off(jr, L) + ir;
#pragma unroll
    for (int c = 0; c < NEQ; ++c) { ql[c] = a[c * L.pitch]; qr[c] = b[c * L.pitch]; }
    prims_fast<S>(ql, (const R*)nullptr, P, pl);
    prims_fast<S>(qr, (const R*)nullptr, P, pr);
    const bool clean = S::cell_ok(ql, (const R*)nullptr, pl, P) &&
                       S::cell_ok(qr, (const R*)nullptr, pr, P);
    if (dir == 0) probe_next<S, R, 1>(ql, qr, pl, pr, clean, P, L, gi, gj, mx, key);
    else probe_next<S, R, 2>(ql, qr, pl, pr, clean, P, L, gi, gj, my, key);
  }
  if (key != ~0ull) atomicMax(&ds->slot[slot][2], NKEY_MAX - key);
  unsigned long long bx = Bits<R>::to(mx), by = Bits<R>::to(my);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long wx = __shfl_xor_sync(0xffffffffu, bx, o);
    unsigned long long wy = __shfl_xor_sync(0xffffffffu, by, o);
    bx = wx > bx ? wx : bx;
    by = wy > by ? wy : by;
  }
  const int lane = tid & 31, wid = tid >> 5;
  if (lane == 0) { sred[0][wid] = bx; sred[1][wid] = by; }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < NT / 32; ++w) {
      bx = sred[0][w] > bx ? sred[0][w] : bx;
      by = sred[1][w] > by ? sred[1][w] : by;
    }
    atomicMax(&ds->slot[slot][0], bx);
    atomicMax(&ds->slot[slot][1], by);
  }
}

// Which tile probes the next pre-pass's lower-bound edges (k_speeds_t): the
// hint edge of each direction (where this step's maximum was found), moved
// by at most one cell so that both of its cells are interior and lie in one
// 29x29 tile.  own = that tile's index (-1: none), off = offset of the lower
// / left cell in it.
__device__ __forceinline__ void hint_owner(unsigned long long hk, const Layout& L, int d,
                                           int& own, int& off) {
  constexpr int LW = 29;
  own = -1; off = 0;
  if (hk == 0ull) return;
  const unsigned idx = (unsigned)(hk & HINT_IDX_MASK);
  const unsigned w = d == 0 ? (unsigned)L.nx + 1u : (unsigned)L.nx;
  const int hj = (int)(idx / w), hi = (int)(idx - (unsigned)hj * w);
  int ci, cj;
  if (d == 0) {
    if (L.nx < 2 || hj >= L.ny) return;
    ci = min(max(hi - 1, 0), L.nx - 2);
    if (ci % LW == LW - 1) ci -= 1;
    cj = hj;
  } else {
    if (L.ny < 2 || hi >= L.nx) return;
    cj = min(max(hj - 1, 0), L.ny - 2);
    if (cj % LW == LW - 1) cj -= 1;
    ci = hi;
  }
  own = (cj / LW) * ((L.nx + LW - 1) / LW) + ci / LW;
  off = (cj % LW) * LW + ci % LW;
}

// one edge per lane of a grid line (see k_update_w): solve, optional
// admissibility probe, wave limiter against lane +-1 (register shuffles),
// correction flux; returns this lane's apdq / flux and the next lane's
// amdq / flux (the right edge of the lane's cell)
template <class S, class R, int ORDER, int LIM, bool CHECKS, int NI, int HC>
__device__ __forceinline__ void line_edge(const R* sQ, const R* sA, const R* sP,
                                          const typename S::template Params<R>& P,
                                          const Layout& L, int cl, int cr, int ei, int ej,
                                          bool ref, R dtdn, unsigned long long& key,
                                          R* ap, R* amn, R* fl, R* fr) {
  constexpr int NEQ = S::NEQ, NW = S::NW, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int NA1 = NAUX > 0 ? NAUX : 1, NP1 = NPR > 0 ? NPR : 1;
  constexpr unsigned FULL = 0xffffffffu;
  R ql[NEQ], qr[NEQ], al[NA1], ar[NA1], pl[NP1], pr[NP1];
#pragma unroll
  for (int c = 0; c < NEQ; ++c) { ql[c] = sQ[c * HC + cl]; qr[c] = sQ[c * HC + cr]; }
#pragma unroll
  for (int c = 0; c < NAUX; ++c) { al[c] = sA[c * HC + cl]; ar[c] = sA[c * HC + cr]; }
#pragma unroll
  for (int c = 0; c < NPR; ++c) { pl[c] = sP[c * HC + cl]; pr[c] = sP[c * HC + cr]; }
  R W[NW][NEQ], s[NW], am[NEQ], apl[NEQ];
  bool oks = true;
  S::template solve<NI, FastMath>(ql, qr, pl, pr, al, ar, P, W, s, am, apl, oks);
  if (!oks) S::template solve<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, W, s, am, apl, oks);
  if (CHECKS && ref) {
    R sm;
    bool okm = true;
    int code = S::template probe<NI, IeeeMath>(ql, qr, pl, pr, al, ar, P, sm, okm);
    if (code) {
      unsigned long long kk = err_key(NI - 1, ei, L.j_off + ej, (code & 0xff) - 1, code >> 8,
                                      L.nx);
      key = kk < key ? kk : key;
    }
  }
  R f[NEQ];
  bool fz[NEQ];
#pragma unroll
  for (int m = 0; m < NEQ; ++m) { f[m] = (R)0; fz[m] = true; }
  if (ORDER == 2) {
    R dupw[NW], doww[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      R dup = (R)0, dow = (R)0;
      bool first = true;
      // upwind edge: lane-1 if s > 0 else lane+1 (one indexed shuffle per value)
      const int src = (s[w] > (R)0) ? (int)(threadIdx.x & 31) - 1 : (int)(threadIdx.x & 31) + 1;
#pragma unroll
      for (int m = 0; m < NEQ; ++m) {
        if (S::template wzero<NI>(w, m)) continue;   // structural zero: no term
        const R up = __shfl_sync(FULL, W[w][m], src & 31);
        dup = first ? up * W[w][m] : dup + up * W[w][m];
        dow = first ? W[w][m] * W[w][m] : dow + W[w][m] * W[w][m];
        first = false;
      }
      dupw[w] = dup;
      doww[w] = dow;
    }
    // the NW limiter ratios as independent FastMath divisions, one fallback
    R thw[NW];
    bool okt = true;
    // LIMSEL: theta = dup / dow, 0 where dow == 0.  dup == +-0 gives theta =
    // +-0 (dow is a sum of squares: positive, and NaN only together with
    // dup), and every limiter maps +-0 to +0: so phi = +0 whenever dup == 0
    // or dow == 0, the quotient is unguarded and its range test only counts
    // otherwise
    constexpr bool LIMSEL = LinePolicy<S, R>::LIMSEL;
    bool spw[NW];
    if constexpr (LIMSEL) {
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        bool okc;
        thw[w] = FastMath::div_core(dupw[w], doww[w], okc);
        spw[w] = (doww[w] == (R)0) || (dupw[w] == (R)0);
        okt = okt && (spw[w] || okc);
      }
    } else {
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const bool nz = doww[w] != (R)0;
        const R q = FastMath::div(nz ? dupw[w] : (R)0, nz ? doww[w] : (R)1, okt);
        thw[w] = nz ? q : (R)0;
        spw[w] = false;
      }
    }
    if (!okt) {
#pragma unroll
      for (int w = 0; w < NW; ++w) thw[w] = (doww[w] != (R)0) ? dupw[w] / doww[w] : (R)0;
    }
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      R th = thw[w];
      R ph = limiter_phi<LIM>(th);
      if (LIMSEL && LIM != LIM_NONE) ph = spw[w] ? (R)0 : ph;
      R a = fabs(s[w]);
      R coef = a * ((R)1 - dtdn * a);
      R cph = coef * ph;
#pragma unroll
      for (int m = 0; m < NEQ; ++m) {
        if (S::template wzero<NI>(w, m)) continue;
        R wl = cph * W[w][m];
        f[m] = fz[m] ? wl : f[m] + wl;
        fz[m] = false;
      }
    }
#pragma unroll
    for (int m = 0; m < NEQ; ++m) f[m] = (R)0.5 * f[m];
  }
#pragma unroll
  for (int m = 0; m < NEQ; ++m) {
    ap[m] = apl[m];
    amn[m] = __shfl_down_sync(FULL, am[m], 1);
    fr[m] = __shfl_down_sync(FULL, f[m], 1);
    fl[m] = f[m];
  }
}

// Staging of an INTERIOR tile (no boundary mapping) for the line kernel, a
// halo row per warp and slot: lane = column 0..31, so a row's address is one
// warp-uniform base plus the lane; column 32 of rows 0..31 goes into the free
// last slot of the last staging warp (cell (32, 32) is one of the halo's
// 2 x 2 corners, which feed no edge).  All of a thread's loads are issued
// before the first is used.  Returns "every staged cell admissible" (CHECKS).
// Not inlined, like band_prefetch: its registers are its own.
template <class S, class R, int NSW, bool CHECKS>
__device__ __noinline__ int stage_inner(const R* __restrict__ q, const R* __restrict__ aux,
                                        R* __restrict__ sQ, long long pitch, long long rstride,
                                        long long astride, int i0, int j0,
                                        const typename S::template Params<R> P) {
  constexpr int NEQ = S::NEQ, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int NA1 = NAUX > 0 ? NAUX : 1, NP1 = NPR > 0 ? NPR : 1;
  constexpr int HW = 33, HC = HW * HW;
  constexpr int NSTG = (HW + NSW - 1) / NSW;
  static_assert(NSW >= 1 && (NSW - 1) + (NSTG - 1) * NSW >= HW, "no free slot for column 32");
  R* sA = sQ + NEQ * HC;
  R* sP = sA + NAUX * HC;
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  auto slot_cell = [&](int k, int& lx, int& ly) {
    lx = lane; ly = warp + k * NSW;
    if (k == NSTG - 1 && warp == NSW - 1) { lx = HW - 1; ly = lane; }
    return ly < HW;
  };
  R qs[NSTG][NEQ], as[NSTG][NA1];
#pragma unroll
  for (int k = 0; k < NSTG; ++k) {
    int lx, ly;
    if (slot_cell(k, lx, ly)) {
      const R* src = q + (long long)(j0 + ly) * rstride + (i0 - 2 + lx);
#pragma unroll
      for (int c = 0; c < NEQ; ++c) qs[k][c] = __ldcg(src + c * pitch);
      if (NAUX > 0) {
        const R* asrc = aux + (long long)(j0 + ly) * astride + (i0 - 2 + lx);
#pragma unroll
        for (int c = 0; c < NAUX; ++c) as[k][c] = __ldcg(asrc + c * pitch);
      }
    }
  }
  bool ok = true;
#pragma unroll
  for (int k = 0; k < NSTG; ++k) {
    int lx, ly;
    if (slot_cell(k, lx, ly)) {
      const int idx = ly * HW + lx;
#pragma unroll
      for (int c = 0; c < NEQ; ++c) sQ[c * HC + idx] = qs[k][c];
#pragma unroll
      for (int c = 0; c < NAUX; ++c) sA[c * HC + idx] = as[k][c];
      R pc[NP1];
      if (NPR > 0) {
        prims_fast<S>(qs[k], as[k], P, pc);
#pragma unroll
        for (int c = 0; c < NPR; ++c) sP[c * HC + idx] = pc[c];
      }
      if (CHECKS) ok = ok && S::cell_ok(qs[k], as[k], pc, P);
    }
  }
  return ok ? 1 : 0;
}

// device-side reduction across shards: wait until every shard pushed its
// slot for this step (release/acquire through the arrival counter)
__device__ __forceinline__ void wait_arrivals(DevState* ds, unsigned long long need) {
  wait_counter(&ds->arrive, need, ds);
}

// --------------------------------------------------------------------------
// Warp-per-line fused update (default for 3-component systems).
//
// Tile = LW x LW cells with LW = 29: one warp's 32 lanes own the 32
// consecutive edges of one grid line that the tile's 29 cells need (their 30
// edges plus the limiter's two outer neighbours).  So:
//   * the wave limiter fetches the upwind neighbour's wave with a register
//     shuffle (lane +-1) instead of a shared-memory round trip;
//   * the next edge's amdq / flux for the cell update is one more shuffle;
//   * each sweep direction is ONE barrier-free pass (x: warps walk rows,
//     y: warps walk columns), 3 barriers per tile in total.
// The x pass leaves q1 = (q - dtdx (apdq_i + amdq_{i+1})) - dtdx (F~_{i+1} - F~_i)
// per cell in shared memory; the y pass subtracts the y term and then the y
// correction (the oracle's dimension-by-dimension order) and writes q_new
// back to shared memory, from which the tile is stored row-coalesced.
template <class S, class R, int ORDER, int LIM, int NWARP, bool CHECKS, bool FUSED,
          bool PERSIST = false>
__global__ void __launch_bounds__(NWARP * 32, ((sizeof(R) == 4 || WS_LB3) && NWARP == 10
                                                   ? (S::NEQ >= 4 ? (sizeof(R) == 8 ? 2 : 3)
                                                      : sizeof(R) == 4 ? WS_F32_MINB : 3)
                                                   : NWARP == 15 && S::NEQ <= 3 ? 2
                                                   : (20 / NWARP > 0 ? 20 / NWARP : 1)))
// (10-warp CTAs: three per SM -- 30 warps, <= 64 registers, <= 75 KB of
// shared memory each; four per SM for fp32 up to 3 components (48
// registers, 36 KB); two for 4-component fp64 (111 KB); WS_LB3=0 builds the
// two-per-SM form for comparison.
// Measured and dropped for 3-component fp64: the persistent prefetching
// form at one 15-warp CTA per SM (-18 %) and at two (-19 % on C5))
k_update_w(const R* __restrict__ q, const R* __restrict__ aux, R* __restrict__ qn,
           const Layout L, const typename S::template Params<R> P, const StepArgs A,
           DevState* __restrict__ ds) {
  constexpr int NEQ = S::NEQ, NW = S::NW, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int LW = 29, HW = 33, HC = HW * HW, NT = NWARP * 32;
  constexpr int NA1 = NAUX > 0 ? NAUX : 1, NP1 = NPR > 0 ? NPR : 1;
  constexpr unsigned FULL = 0xffffffffu;
  // per-tile accumulators for the next tile pre-pass (S::tile_acc): not in
  // the checked (static-speed single-domain) and fused forms, which have none
  constexpr bool TILES = HasTile<S>::value && !FUSED && !CHECKS;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sQ = reinterpret_cast<R*>(smem_raw);
  R* sA = sQ + NEQ * HC;
  R* sP = sA + NAUX * HC;
  R* sX = sP + NPR * HC;          // [NEQ][LW*LW]: q1 after the x pass, later q_new
                                  // (FUSED: [2*NEQ], the next state's prims after it)
  R* sR = sX + (FUSED ? 2 : 1) * NEQ * LW * LW;  // PERSIST: raw q (+aux) of the next tile
  static_assert(!(PERSIST && FUSED), "persistent form has no fused epilogue");

  // warp index through a lane-0 broadcast: the compiler then treats it as
  // warp-uniform, so the line loops below (trip count depends on it) keep
  // their shuffles plain instead of divergent-warp collectives
  const int tid = threadIdx.x, lane = tid & 31, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  // one thread evaluates the step control (dt from this step's maxima, 5
  // dependent divisions) while the others stage the tile; the result is
  // handed over at the post-staging barrier
  __shared__ Ctl s_ctl;
  __shared__ R s_dtd[2];
  __shared__ int s_hown[2], s_hoff[2];  // TMAX: tile holding the hint edge (-1: none), offset
  __shared__ int s_acc[NAcc<S>::value][NWARP];  // TMAX: per-warp S::tile_acc of the tile
  // PERSIST (one CTA per SM, 4-component fp64): CTAs walk the tiles and
  // prefetch the next tile's raw state with cp.async while the current tile
  // computes; otherwise one tile per CTA (blockIdx)
  const int ntx = (L.nx + LW - 1) / LW, nty = (L.ny + LW - 1) / LW, ntiles = ntx * nty;
  // row-strip overlap (ws_phase_update_part): part 1 = the boundary tile
  // rows [0, tr_lo) and [tr_hi, nty) -- every cell a neighbour needs as a
  // ghost row --, part 2 = the interior tile rows [tr_lo, tr_hi), launched
  // while the new boundary rows travel; v indexes the tiles of the part
  const int nvt = ntx * (A.part == 0 ? nty : A.part == 1 ? A.tr_lo + nty - A.tr_hi
                                                         : A.tr_hi - A.tr_lo);
  auto vtile = [&](int vv) {
    int ty = vv / ntx;
    const int tx = vv - ty * ntx;
    if (A.part == 1) { if (ty >= A.tr_lo) ty += A.tr_hi - A.tr_lo; }
    else if (A.part == 2) ty += A.tr_lo;
    return ty * ntx + tx;
  };
  // part row -> tile row (vtile's row mapping)
  auto vrow = [&](int ty) {
    if (A.part == 1) { if (ty >= A.tr_lo) ty += A.tr_hi - A.tr_lo; }
    else if (A.part == 2) ty += A.tr_lo;
    return ty;
  };
  int v = PERSIST ? (int)blockIdx.x : (int)(blockIdx.y * gridDim.x + blockIdx.x);
  auto tile_origin = [&](int tt, int& a, int& b) { a = (tt % ntx) * LW; b = (tt / ntx) * LW; };
  // raw tile + halo -> sR (BC by index mapping), one cp.async group
  auto prefetch = [&](int tt) {
    int a, b;
    tile_origin(tt, a, b);
    const bool in = a >= 2 && a + LW + 2 <= L.nx && b >= 2 && b + LW + 2 <= L.ny;
    for (int idx = tid; idx < HC; idx += NT) {
      const int lx = idx % HW, ly = idx / HW;
      int gi = a - 2 + lx, gj = b - 2 + ly;
      if (!in) { gi = map_i(gi, L); gj = map_j(gj, L); }
      WS_CHK(L, gi >= 0 && gi < L.nx && row_readable(gj, L), CHK_STAGE_READ);
      const R* src = q + row_off(gj, L) + gi;
#pragma unroll
      for (int c = 0; c < NEQ; ++c) cp_async(&sR[c * HC + idx], src + c * L.pitch);
      if (NAUX > 0) {
        const R* asrc = aux + (long long)(gj + 2) * L.astride + gi;
#pragma unroll
        for (int c = 0; c < NAUX; ++c) cp_async(&sR[(NEQ + c) * HC + idx], asrc + c * L.pitch);
      }
    }
    cp_commit();
  };
  // one tile per CTA: the grid is (ntx, part rows), so the tile's column and
  // part row are the block indices themselves (no division by ntx)
  int t, i0, j0;
  if (PERSIST) {
    t = vtile(v);
    tile_origin(t, i0, j0);
  } else {
    const int ty = vrow((int)blockIdx.y);
    t = ty * ntx + (int)blockIdx.x;
    i0 = (int)blockIdx.x * LW;
    j0 = ty * LW;
  }
  Ctl ctl;
  bool stage_ok = true;   // CHECKS: every staged cell admissible (per thread)
  const unsigned long long t_start = L.trace ? gtimer() : 0ull;
  // PDL: the next step's pre-pass may launch once every CTA of this grid has
  // started (it waits for this grid's completion before reading anything).
  // With a pre-pass in front (!CHECKS), the tile staging below reads only the
  // state of the PREVIOUS update, which had completed before the pre-pass
  // triggered this launch, so only the thread reading the pre-pass's maxima
  // waits; without one (CHECKS: static speeds) everyone waits first.
  pdl_trigger();
  if (CHECKS) pdl_wait();
  if (PERSIST) {
    if (v < nvt) prefetch(t);
    if (tid == NT - 32) {
      if (!CHECKS) pdl_wait();
      if (!CHECKS && L.npeers > 0) wait_arrivals(ds, (unsigned long long)L.npeers * (unsigned long long)(__ldcg(&ds->seq) + 1));
      const Ctl c0 = step_control<R>(A, ds, !CHECKS);
      s_ctl = c0;
      s_dtd[0] = (R)(c0.dt / A.dx);
      s_dtd[1] = (R)(c0.dt / A.dy);
    }
  }
  // TMAX (tile pre-pass): after the tile's warps reduced into s_acc and the
  // new tile sits in sX: warp 0 folds and stores the tile accumulators, the
  // tile that holds a hint edge probes it (the next pre-pass's exact lower
  // bound).  Runs after a barrier that follows the tile's store loop.
  int t_prev = -1;
  auto finish_tile = [&](int tt) {
    if constexpr (TILES) {
    constexpr int NA = NAcc<S>::value;
    constexpr unsigned MINS = AccMin<S>::value;
    if (tid < NA) {
      // lane k of warp 0 folds slot k over the warps and stores it
      const bool mn = (MINS >> tid) & 1u;
      int v = s_acc[tid][0];
#pragma unroll
      for (int w = 1; w < NWARP; ++w) v = mn ? min(v, s_acc[tid][w]) : max(v, s_acc[tid][w]);
      static_cast<int*>(A.tmax)[((long long)(A.cur ^ 1) * ntiles + tt) * NA + tid] = v;
    }
    // (static speeds: no hint edge, its probe would need aux)
    if (!S::STATIC_SPEEDS && (tid == 0 || tid == 32)) {
      const int d = tid >> 5;
      const int o = s_hown[d] == tt ? s_hoff[d] : -1;
      if (o >= 0) {
        R ql[NEQ], qr[NEQ], pl[NP1], pr[NP1];
        const int o2 = d == 0 ? o + 1 : o + LW;
#pragma unroll
        for (int m = 0; m < NEQ; ++m) { ql[m] = sX[m * (LW * LW) + o]; qr[m] = sX[m * (LW * LW) + o2]; }
        R sm = (R)0;
        if (NPR > 0) { prims_fast<S>(ql, (const R*)nullptr, P, pl); prims_fast<S>(qr, (const R*)nullptr, P, pr); }
        if (S::cell_ok(ql, (const R*)nullptr, pl, P) && S::cell_ok(qr, (const R*)nullptr, pr, P)) {
          bool ok = true;
          int code;
          if (d == 0) {
            code = S::template probe_fast<1, FastMath>(ql, qr, pl, pr, (const R*)nullptr, (const R*)nullptr, P, sm, ok);
            if (!ok) code = S::template probe_fast<1, IeeeMath>(ql, qr, pl, pr, (const R*)nullptr, (const R*)nullptr, P, sm, ok);
          } else {
            code = S::template probe_fast<2, FastMath>(ql, qr, pl, pr, (const R*)nullptr, (const R*)nullptr, P, sm, ok);
            if (!ok) code = S::template probe_fast<2, IeeeMath>(ql, qr, pl, pr, (const R*)nullptr, (const R*)nullptr, P, sm, ok);
          }
          if (code) sm = (R)0;
        }
        ds->tnext[A.cur ^ 1][d] = Bits<R>::to(sm);
      }
    }
    }
  };
  for (;;) {
  if (PERSIST) {
    if (v >= nvt) break;
    cp_wait<0>();
    __syncthreads();   // raw tile landed for every thread; previous tile fully stored
    if constexpr (TILES) {
      if (A.tmax && t_prev >= 0) finish_tile(t_prev);
    }
    stage_ok = true;   // CHECKS: per tile
#pragma unroll 4
    for (int idx = tid; idx < HC; idx += NT) {
      R qc[NEQ], ac[NA1], pc[NP1];
#pragma unroll
      for (int c = 0; c < NEQ; ++c) { qc[c] = sR[c * HC + idx]; sQ[c * HC + idx] = qc[c]; }
#pragma unroll
      for (int c = 0; c < NAUX; ++c) { ac[c] = sR[(NEQ + c) * HC + idx]; sA[c * HC + idx] = ac[c]; }
      if (NPR > 0) {
        prims_fast<S>(qc, ac, P, pc);
#pragma unroll
        for (int c = 0; c < NPR; ++c) sP[c * HC + idx] = pc[c];
      }
      if (CHECKS) stage_ok = stage_ok && S::cell_ok(qc, ac, pc, P);
    }
    __syncthreads();   // sR consumed: the next tile's copies may land
    if (v + (int)gridDim.x < nvt) prefetch(vtile(v + (int)gridDim.x));
  } else {
    // ---- stage tile + 2-cell halo (BC by index mapping), per-cell primitives
    const bool inner = i0 >= 2 && i0 + LW + 2 <= L.nx && j0 >= 2 && j0 + LW + 2 <= L.ny;
    // step control by lane 0 of the last warp
    auto do_ctl = [&]() {
      if (!CHECKS) pdl_wait();
      if (!CHECKS && L.npeers > 0) wait_arrivals(ds, (unsigned long long)L.npeers * (unsigned long long)(__ldcg(&ds->seq) + 1));
      const Ctl c0 = step_control<R>(A, ds, !CHECKS);
      s_ctl = c0;
      s_dtd[0] = (R)(c0.dt / A.dx);
      s_dtd[1] = (R)(c0.dt / A.dy);
    };
    constexpr bool FASTSTAGE = LinePolicy<S, R>::FASTSTAGE && NWARP >= 4 && !WS_CHECKED;
    if (FASTSTAGE && inner) {
      // interior tile: warps 0 .. NWARP-2 stage it (stage_inner), the last
      // warp prefetches the band further down and evaluates the step control
      if (warp == NWARP - 1) {
        if constexpr (WS_L2PF != 0) {
          if (lane == 1) {
            const int tyv = (int)blockIdx.y, txv = (int)blockIdx.x;
            const int ka = (WS_PFD + ntx - 1) / ntx;
            if (tyv + ka < (int)gridDim.y)
              band_prefetch<R, NEQ, NAUX, HW>(q, aux, L.nx, L.ny, L.pitch, L.rstride, L.astride,
                                              ntx, txv, vrow(tyv + ka) * LW - 2);
          }
        }
        if (lane == 0) do_ctl();
      } else {
        stage_ok = stage_inner<S, R, NWARP - 1, CHECKS>(q, aux, sQ, L.pitch, L.rstride, L.astride,
                                                        i0, j0, P) != 0;
      }
    } else {
    // all of this thread's loads first (NSTG cells in flight), then the
    // primitives: the loads' latency is paid once per tile, not per cell.
    // L2 loads (ld.global.cg): this grid may have launched before the
    // pre-pass finished, so nothing is taken from a possibly stale L1 line
    // ROWSTAGE: a halo row per warp and slot (lane = column 0..31: the
    // row's address is warp-uniform, the shared-memory index row * HW +
    // lane); column 32 of rows 0..31 in the free last slot of warp NWARP-2.
    // The halo's four 2 x 2 corners feed no edge, so the one cell left over
    // (32, 32) is not staged at all.
    constexpr bool ROWSTAGE = LinePolicy<S, R>::ROWSTAGE;
    constexpr int NSTG = ROWSTAGE ? (HW + NWARP - 1) / NWARP : (HC + NT - 1) / NT;
    static_assert(!ROWSTAGE || (NWARP >= 2 && (NWARP - 2) + (NSTG - 1) * NWARP >= HW),
                  "no free slot for column 32");
    auto slot_cell = [&](int k, int& lx, int& ly) {
      if constexpr (ROWSTAGE) {
        lx = lane; ly = warp + k * NWARP;
        if (k == NSTG - 1 && warp == NWARP - 2) { lx = HW - 1; ly = lane; }
        return ly < HW;
      } else {
        const int idx = tid + k * NT;
        lx = idx % HW; ly = idx / HW;
        return idx < HC;
      }
    };
    if constexpr (WS_L2PF != 0) {
      // Band prefetch (band_prefetch above), by one thread before the tile's
      // own loads
      if (tid == 32) {
        const int tyv = (int)blockIdx.y, txv = (int)blockIdx.x;
        const int ka = (WS_PFD + ntx - 1) / ntx;
        if (tyv + ka < (int)gridDim.y)
          band_prefetch<R, NEQ, NAUX, HW>(q, aux, L.nx, L.ny, L.pitch, L.rstride, L.astride, ntx,
                                          txv, vrow(tyv + ka) * LW - 2);
      }
    }
    // loads in batches of SB cells per thread (LinePolicy::STGB)
    constexpr int SB = LinePolicy<S, R>::STGB > 0 && LinePolicy<S, R>::STGB < NSTG
                           ? LinePolicy<S, R>::STGB : NSTG;
#pragma unroll
    for (int k0 = 0; k0 < NSTG; k0 += SB) {
    R qs[SB][NEQ], as[SB][NA1];
#pragma unroll
    for (int kk = 0; kk < SB; ++kk) {
      int lx, ly;
      if (k0 + kk < NSTG && slot_cell(k0 + kk, lx, ly)) {
        int gi = i0 - 2 + lx, gj = j0 - 2 + ly;
        if (!inner) { gi = map_i(gi, L); gj = map_j(gj, L); }
        WS_CHK(L, gi >= 0 && gi < L.nx && row_readable(gj, L), CHK_STAGE_READ);
        const R* src = q + row_off(gj, L) + gi;
#pragma unroll
        for (int c = 0; c < NEQ; ++c) qs[kk][c] = __ldcg(src + c * L.pitch);
        if (NAUX > 0) {
          const R* asrc = aux + (long long)(gj + 2) * L.astride + gi;
#pragma unroll
          for (int c = 0; c < NAUX; ++c) as[kk][c] = __ldcg(asrc + c * L.pitch);
        }
      }
    }
    // step control by lane 0 of the last warp (one staged cell fewer than
    // the first warps) while its loads are in flight
    if (k0 == 0 && tid == NT - 32) do_ctl();
#pragma unroll
    for (int kk = 0; kk < SB; ++kk) {
      int lx, ly;
      if (k0 + kk < NSTG && slot_cell(k0 + kk, lx, ly)) {
        const int idx = ly * HW + lx;
#pragma unroll
        for (int c = 0; c < NEQ; ++c) sQ[c * HC + idx] = qs[kk][c];
#pragma unroll
        for (int c = 0; c < NAUX; ++c) sA[c * HC + idx] = as[kk][c];
        R pc[NP1];
        if (NPR > 0) {
          prims_fast<S>(qs[kk], as[kk], P, pc);
#pragma unroll
          for (int c = 0; c < NPR; ++c) sP[c * HC + idx] = pc[c];
        }
        if (CHECKS) stage_ok = stage_ok && S::cell_ok(qs[kk], as[kk], pc, P);
      }
    }
    }   // batches
    }   // boundary-mapped staging
  }
  // CHECKS (static speeds, no pre-pass): a tile whose staged cells are all
  // admissible cannot report an error, so its edges skip the checked probe
  const bool tile_clean = CHECKS ? (__syncthreads_and(stage_ok) != 0) : (__syncthreads(), true);
  ctl = s_ctl;
  if (ctl.skip) break;
  {
    const R dtdx = s_dtd[0];
    const R dtdy = s_dtd[1];
    unsigned long long key = ~0ull;

    const bool cell_lane = lane >= 1 && lane <= LW;

    // TMAX: the last warp walks one row fewer in the x pass; during a CTA's
    // first tile it fetches and decodes this step's hint edges (the pre-pass
    // has completed: the step-control thread waited for it before the
    // barrier above)
    unsigned long long hk0 = 0ull;
    const bool hwarp = TILES && A.tmax != nullptr && t_prev < 0 &&
                       warp == NWARP - 1 && lane < 2;
    if (hwarp) hk0 = __ldcg(&ds->hint_acc[A.cur][lane]);
    // ---- x pass: warps walk rows; lane l = x-edge i0-1+l
    for (int r = warp; r < LW; r += NWARP) {
      if (j0 + r >= L.ny) break;
      const int cl = (r + 2) * HW + lane, cr = cl + 1;
      WS_CHK(L, cl >= 0 && cr < HC, CHK_EDGE_SMEM);
      const int ei = i0 - 1 + lane;
      R ap[NEQ], amn[NEQ], fl[NEQ], fr[NEQ];
      line_edge<S, R, ORDER, LIM, CHECKS, 1, HC>(sQ, sA, sP, P, L, cl, cr, ei, j0 + r,
                                                  !tile_clean && lane >= 1 && lane <= 30 &&
                                                      ei <= L.nx,
                                                  dtdx, key, ap, amn, fl, fr);
      if (cell_lane) {
        const int c = lane - 1;
#pragma unroll
        for (int m = 0; m < NEQ; ++m) {
          const R qc = sQ[m * HC + cr];
          R v = qc - dtdx * (ap[m] + amn[m]);
          if (ORDER == 2) v = v - dtdx * (fr[m] - fl[m]);
          WS_CHK(L, r * LW + c < LW * LW, CHK_X_SMEM);
          sX[m * (LW * LW) + r * LW + c] = v;
        }
      }
    }
    if (hwarp) {
      int own, off;
      hint_owner(hk0, L, lane, own, off);
      s_hown[lane] = own; s_hoff[lane] = off;
    }
    __syncthreads();

    // ---- y pass: warps walk columns; lane l = y-edge j0-1+l
    const int nxv = min(LW, L.nx - i0), nyv = min(LW, L.ny - j0);
    R nmx = (R)0, nmy = (R)0;             // FUSED: next state's max |s|
    unsigned long long nkey = ~0ull;      // FUSED: next state's first bad edge
    for (int c = warp; c < LW; c += NWARP) {
      if (i0 + c >= L.nx) break;
      const int cl = lane * HW + c + 2, cr = cl + HW;
      WS_CHK(L, cl >= 0 && cr < HC, CHK_EDGE_SMEM);
      const int ej = j0 - 1 + lane;
      R ap[NEQ], amn[NEQ], fl[NEQ], fr[NEQ];
      line_edge<S, R, ORDER, LIM, CHECKS, 2, HC>(sQ, sA, sP, P, L, cl, cr, i0 + c, ej,
                                                  !tile_clean && lane >= 1 && lane <= 30 &&
                                                      ej < L.ny_edges_y,
                                                  dtdy, key, ap, amn, fl, fr);
      R qnew[NEQ];
      const int rr = lane - 1, o = rr * LW + c;
      WS_CHK(L, !cell_lane || (o >= 0 && o < LW * LW), CHK_X_SMEM);
      if (cell_lane) {
#pragma unroll
        for (int m = 0; m < NEQ; ++m) {
          R v = sX[m * (LW * LW) + o] - dtdy * (ap[m] + amn[m]);
          if (ORDER == 2) v = v - dtdy * (fr[m] - fl[m]);
          sX[m * (LW * LW) + o] = v;
          qnew[m] = v;
        }
      }
      if (FUSED) {
        // the next state's primitives (kept in the consumed dFx slots) and its
        // y-edges inside this tile column: the lower cell is lane - 1
        static_assert(!FUSED || (NPR <= NEQ && NAUX == 0), "FUSED epilogue layout");
        R pn[NP1];
        bool cok = false;
        if (cell_lane) {
          prims_fast<S>(qnew, (const R*)nullptr, P, pn);
#pragma unroll
          for (int k = 0; k < NPR; ++k) sX[(NEQ + k) * (LW * LW) + o] = pn[k];
          cok = S::cell_ok(qnew, (const R*)nullptr, pn, P);
        } else {
#pragma unroll
          for (int m = 0; m < NEQ; ++m) qnew[m] = (R)1;
#pragma unroll
          for (int k = 0; k < NPR; ++k) pn[k] = (R)1;
        }
        R ql[NEQ], pl[NP1];
#pragma unroll
        for (int m = 0; m < NEQ; ++m) ql[m] = __shfl_up_sync(0xffffffffu, qnew[m], 1);
#pragma unroll
        for (int k = 0; k < NPR; ++k) pl[k] = __shfl_up_sync(0xffffffffu, pn[k], 1);
        const bool okl = __shfl_up_sync(0xffffffffu, cok, 1);
        const int gj = j0 + rr;
        if (cell_lane && rr < nyv) {
          if (rr >= 1)
            probe_next<S, R, 2>(ql, qnew, pl, pn, okl && cok, P, L, i0 + c, gj, nmy, nkey);
          if (rr == 0 && gj == 0 && L.bcy != BC_PERIODIC)
            probe_next<S, R, 2>(qnew, qnew, pn, pn, cok, P, L, i0 + c, 0, nmy, nkey);
          if (rr == nyv - 1 && gj + 1 == L.ny && L.bcy != BC_PERIODIC)
            probe_next<S, R, 2>(qnew, qnew, pn, pn, cok, P, L, i0 + c, L.ny, nmy, nkey);
        }
      }
    }
    __syncthreads();

    if (FUSED) {
      // x-edges inside each tile row of the next state: lane l = cell l
      for (int r = warp; r < LW; r += NWARP) {
        if (r >= nyv) break;
        const int l = lane < LW ? lane : LW - 1;
        const int o = r * LW + l;
        R qc[NEQ], pc[NP1], ql[NEQ], pl[NP1];
#pragma unroll
        for (int m = 0; m < NEQ; ++m) qc[m] = sX[m * (LW * LW) + o];
#pragma unroll
        for (int k = 0; k < NPR; ++k) pc[k] = sX[(NEQ + k) * (LW * LW) + o];
        const bool cok = S::cell_ok(qc, (const R*)nullptr, pc, P);
#pragma unroll
        for (int m = 0; m < NEQ; ++m) ql[m] = __shfl_up_sync(0xffffffffu, qc[m], 1);
#pragma unroll
        for (int k = 0; k < NPR; ++k) pl[k] = __shfl_up_sync(0xffffffffu, pc[k], 1);
        const bool okl = __shfl_up_sync(0xffffffffu, cok, 1);
        const int gj = j0 + r, gi = i0 + lane;
        if (lane < nxv) {
          if (lane >= 1)
            probe_next<S, R, 1>(ql, qc, pl, pc, okl && cok, P, L, gi, gj, nmx, nkey);
          if (lane == 0 && gi == 0 && L.bcx != BC_PERIODIC)
            probe_next<S, R, 1>(qc, qc, pc, pc, cok, P, L, 0, gj, nmx, nkey);
          if (lane == nxv - 1 && gi + 1 == L.nx && L.bcx != BC_PERIODIC)
            probe_next<S, R, 1>(qc, qc, pc, pc, cok, P, L, L.nx, gj, nmx, nkey);
        }
      }
      // CTA reduction of the next state's maxima into the other slot
      __shared__ unsigned long long s_red2[2][NWARP];
      unsigned long long bx = Bits<R>::to(nmx), by = Bits<R>::to(nmy);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        unsigned long long wx = __shfl_xor_sync(0xffffffffu, bx, off);
        unsigned long long wy = __shfl_xor_sync(0xffffffffu, by, off);
        bx = wx > bx ? wx : bx;
        by = wy > by ? wy : by;
      }
      if (lane == 0) { s_red2[0][warp] = bx; s_red2[1][warp] = by; }
      if (nkey != ~0ull) atomicMax(&ds->slot[A.cur ^ 1][2], NKEY_MAX - nkey);
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < NWARP; ++w) {
          bx = s_red2[0][w] > bx ? s_red2[0][w] : bx;
          by = s_red2[1][w] > by ? s_red2[1][w] : by;
        }
        atomicMax(&ds->slot[A.cur ^ 1][0], bx);
        atomicMax(&ds->slot[A.cur ^ 1][1], by);
      }
    }

    int tb[NAcc<S>::value];   // TMAX: this thread's S::tile_acc accumulator
    if constexpr (TILES) S::acc_init(tb);
    // ---- row-coalesced store of the tile; the strip's two first / last rows
    // also go straight into the low / high neighbour's ghost rows (P2P
    // stores into its buffer of the same parity) when halos are pushed
    const int par = A.cur ^ 1;
    // ROWSTORE: a tile row per warp (lane = column), so the row address and
    // the halo-push tests are warp-uniform; else threads walk the tile's
    // cells linearly
    constexpr bool ROWSTORE = LinePolicy<S, R>::ROWSTORE;
    for (int it = ROWSTORE ? warp : tid; it < (ROWSTORE ? LW : LW * LW); it += ROWSTORE ? NWARP : NT) {
      const int rr = ROWSTORE ? it : it / LW, c = ROWSTORE ? lane : it % LW;
      const int idx = ROWSTORE ? rr * LW + (lane < LW ? lane : 0) : it;
      const int gi = i0 + c, gj = j0 + rr;
      if (c < LW && gi < L.nx && gj < L.ny) {
        R* dst = qn + row_off(gj, L) + gi;
#pragma unroll
        for (int m = 0; m < NEQ; ++m) dst[m * L.pitch] = sX[m * (LW * LW) + idx];
        WS_CHK(L, gi >= 0 && gj >= 0, CHK_STORE);
        if (WS_CHECKED && L.chk) atomicAdd(&L.chk[1 + (long long)gj * L.nx + gi], 1u);
        if constexpr (TILES) {
          // tile-bound ingredients of the new cell for the next pre-pass
          // (k_speeds_t)
          if (A.tmax) {
            R qv[NEQ];
#pragma unroll
            for (int m = 0; m < NEQ; ++m) qv[m] = sX[m * (LW * LW) + idx];
            S::tile_acc(qv, P, tb);
          }
        }
        if (L.nds_lo && gj < 2) {
          R* rd = static_cast<R*>(L.nq_lo[par]) + (long long)(L.ny_lo + 2 + gj) * L.rstride + gi;
#pragma unroll
          for (int m = 0; m < NEQ; ++m) rd[m * L.pitch] = sX[m * (LW * LW) + idx];
        }
        if (L.nds_hi && gj >= L.ny - 2) {
          R* rd = static_cast<R*>(L.nq_hi[par]) + (long long)(gj - (L.ny - 2)) * L.rstride + gi;
#pragma unroll
          for (int m = 0; m < NEQ; ++m) rd[m * L.pitch] = sX[m * (LW * LW) + idx];
        }
      }
    }
    if constexpr (TILES) {
      if (A.tmax) {
        constexpr unsigned MINS = AccMin<S>::value;
#pragma unroll
        for (int k = 0; k < NAcc<S>::value; ++k) {
          const bool mn = (MINS >> k) & 1u;
          const int r = mn ? __reduce_min_sync(FULL, tb[k]) : __reduce_max_sync(FULL, tb[k]);
          if (lane == 0) s_acc[k][warp] = r;
        }
      }
    }
    if ((L.nds_lo && j0 < 2) || (L.nds_hi && j0 + LW > L.ny - 2)) {
      // boundary tile: once every such tile of a side stored, release the
      // neighbour (system fence, then one increment of its arrival counter)
      __syncthreads();
      if (tid == 0) {
        __threadfence_system();
        const int ntxl = (L.nx + LW - 1) / LW;
        if (L.nds_lo && j0 < 2 && atomicAdd(&ds->hsent[0], 1) == ntxl - 1) {
          ds->hsent[0] = 0;
          atomicAdd_system(&L.nds_lo->harrive, 1ull);
        }
        if (L.nds_hi && j0 + LW > L.ny - 2) {
          const int rows = ((L.ny - 1) / LW != (L.ny - 2) / LW) ? 2 : 1;   // tile rows holding ny-2, ny-1
          if (atomicAdd(&ds->hsent[1], 1) == rows * ntxl - 1) {
            ds->hsent[1] = 0;
            atomicAdd_system(&L.nds_hi->harrive, 1ull);
          }
        }
      }
    }
    if (CHECKS && key != ~0ull) atomicMax(&ds->slot[A.cur][2], NKEY_MAX - key);
  }
  t_prev = t;
  if (!PERSIST) break;
  v += gridDim.x;
  t = vtile(v);
  tile_origin(t, i0, j0);
  }   // tile loop
  if (PERSIST) cp_wait<0>();   // no copy outstanding at exit
  __syncthreads();
  ctl = s_ctl;
  if constexpr (TILES) {
    if (A.tmax && !ctl.skip && t_prev >= 0) finish_tile(t_prev);
  }


  // ---- last CTA commits the step.  The fence only orders this CTA's
  // error-key atomics (CHECKS) before its count; the state stores need none
  // (the next kernel reads them after this grid completes), and a fence per
  // CTA holds the SM's slot for its whole latency.
  __syncthreads();
  if (tid == 0) {
    if (CHECKS) __threadfence();
    // a split step (part 1 + part 2) counts the CTAs of both launches
    const int nblk = A.nblk_total > 0 ? A.nblk_total : (int)(gridDim.x * gridDim.y);
    const int prev = atomicAdd(&ds->done, 1);
    if (prev == nblk - 1) {
      __threadfence();
      if constexpr (HasBound<S>::value && !FUSED) {
        if (A.tmax) {
          if (!ctl.skip && s_hown[0] < 0) ds->tnext[A.cur ^ 1][0] = 0ull;
          if (!ctl.skip && s_hown[1] < 0) ds->tnext[A.cur ^ 1][1] = 0ull;
        }
      }
      commit_step<R>(ds, A, ctl, L);
    }
    if (L.trace) trace_cta(L, 1, t_start);
  }
}

// --------------------------------------------------------------------------
// Multi-step form for small grids whose wave speeds are static (acoustics,
// advection: no CFL pre-pass): ONE cooperative launch runs up to nsteps
// steps, one CTA per tile (ntiles <= co-resident CTAs), so a step costs one
// grid barrier instead of one kernel launch (BASELINE C1: 256^2, 81 tiles).
// NWARP = 30: warps 0..28 own one line of the tile in each pass and stage /
// store the tile; the last warp evaluates the step control and records the
// previous step (report, t, counters) while the others work, so neither sits
// on the critical path.  Every CTA derives the same controls from the same
// values (static speeds, t advanced by the same fp64 additions as the
// record), and learns whether an edge of the step was inadmissible from the
// barrier word.  The arithmetic per cell is k_update_w's (line_edge, the
// same update expressions): bitwise the same steps.
//
// Grid barrier: one 64-bit word per step parity, arrivals in the low half,
// arrivals that found an inadmissible edge in the high half, added with one
// release atomic per CTA; a CTA waits (acquire loads) until all arrivals of
// the step are in.  The next use of a parity's word comes two steps later,
// after a barrier every CTA must pass, so its high half is this step's.
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_add_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

// step_control with the static speeds, sticky error and t held by the caller
__device__ __forceinline__ Ctl step_control_local(const StepArgs& A, double msx, double msy,
                                                  double t, int err) {
  Ctl c;
  c.skip = 0; c.stationary = 0; c.finished = 0; c.dt = 0.0; c.msx = msx; c.msy = msy;
  if (err) { c.skip = 1; c.msx = c.msy = 0.0; return c; }
  double remaining = A.remaining;
  int has_rem = A.has_remaining;
  if (A.has_t_final) {
    if (!(A.t_final - t > A.tol)) { c.skip = 1; c.finished = 1; return c; }
    remaining = A.t_final - t;
    has_rem = 1;
  }
  double dt;
  if (A.has_fixed) {
    dt = A.fixed_dt;
  } else {
    double rate = msx / A.dx + msy / A.dy;
    if (rate == 0.0) { c.stationary = 1; c.skip = 1; return c; }
    dt = A.cfl / rate;
  }
  if (A.has_dt_max) dt = (A.dt_max < dt) ? A.dt_max : dt;
  if (has_rem) dt = (remaining < dt) ? remaining : dt;
  c.dt = dt;
  return c;
}

// the control thread's copy of the device counters (only it writes them)
struct RunCtl {
  double t, msx, msy;
  long long steps, nrep, seq;
  int err;
  Ctl pend;          // CTA 0: the applied step still to be recorded
  int pend_cur, have_pend;
  unsigned a0[2], e0[2], uses[2];   // thread 0: barrier words at launch, uses per parity
};

#ifndef WS_RS_PROF
#define WS_RS_PROF 0
#endif

template <class S, class R, int ORDER, int LIM, int NWARP>
__global__ void __launch_bounds__(NWARP * 32, 1)
k_run_small(R* __restrict__ q0, R* __restrict__ q1, const R* __restrict__ aux, const Layout L,
            const typename S::template Params<R> P, const StepArgs A, const int nsteps,
            DevState* __restrict__ ds) {
  constexpr int NEQ = S::NEQ, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int LW = 29, HW = 33, HC = HW * HW, NTW = (NWARP - 1) * 32;
  constexpr int NA1 = NAUX > 0 ? NAUX : 1, NP1 = NPR > 0 ? NPR : 1;
  static_assert(NWARP - 1 >= LW, "one line per working warp");
  static_assert(S::STATIC_SPEEDS, "static wave speeds only (no CFL pre-pass)");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sQ = reinterpret_cast<R*>(smem_raw);
  R* sA = sQ + NEQ * HC;
  R* sP = sA + NAUX * HC;
  R* sX = sP + NPR * HC;          // [NEQ][LW*LW]: q1 after the x pass, then q_new
  __shared__ Ctl s_ctl;
  __shared__ R s_dtd[2];
  __shared__ int s_err;           // 1: an edge of the step was inadmissible; 2: barrier timeout
  __shared__ RunCtl rc;

  const int tid = threadIdx.x, lane = tid & 31, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const bool ctl_warp = warp == NWARP - 1;
  const bool ctl_thr = ctl_warp && lane == 0;
  const bool rec = ctl_thr && blockIdx.x == 0;    // the thread that records the steps
  const int ntx = (L.nx + LW - 1) / LW;
  const int i0 = ((int)blockIdx.x % ntx) * LW, j0 = ((int)blockIdx.x / ntx) * LW;
  const bool inner = i0 >= 2 && i0 + LW + 2 <= L.nx && j0 >= 2 && j0 + LW + 2 <= L.ny;
  const bool cell_lane = lane >= 1 && lane <= LW;
  const unsigned nblk = gridDim.x;
#if WS_RS_PROF
  const bool prof = L.trace && blockIdx.x == 0 && tid == 0;
  auto stamp = [&](int st, int k) {
    if (prof && st * 6 + k < 8 * L.trace_cap) L.trace[st * 6 + k] = gtimer();
  };
#else
  auto stamp = [](int, int) {};
#endif

  if (ctl_thr) {
    // values the previous kernel in the stream committed
    rc.t = __ldcg(&ds->t);
    rc.msx = (double)Bits<R>::from(__ldcg(&ds->static_bits[0]));
    rc.msy = (double)Bits<R>::from(__ldcg(&ds->static_bits[1]));
    rc.steps = __ldcg(&ds->steps);
    rc.nrep = __ldcg(&ds->nrep);
    rc.seq = __ldcg(&ds->seq);
    rc.err = __ldcg(&ds->err);
    rc.have_pend = 0;
  }
  if (tid == 0) {
    for (int p = 0; p < 2; ++p) {
      const unsigned long long w = __ldcg(&ds->mctr[p]);
      rc.a0[p] = (unsigned)w; rc.e0[p] = (unsigned)(w >> 32); rc.uses[p] = 0u;
    }
  }
  // commit_step for one step of this kernel (recording thread only)
  auto record = [&](const Ctl& c, int cur, int errbit) {
    if (rc.err == 0) {
      if (c.finished) {
        ds->finished = 1;
      } else if (errbit) {
        const unsigned long long nk = __ldcg(&ds->slot[cur][2]);
        ds->err_key = NKEY_MAX - nk; ds->err_step = rc.steps; ds->err = ERR_KERNEL;
        rc.err = ERR_KERNEL;
      } else if (c.stationary) {
        ds->err_step = rc.steps; ds->err = ERR_STATIONARY;
        rc.err = ERR_STATIONARY;
      } else {
        Report r;
        r.dt = c.dt;
        r.cfl = c.dt * (c.msx / A.dx + c.msy / A.dy);   // cfl, driver.py:221
        r.msx = c.msx; r.msy = c.msy;
        ds->rep[rc.nrep % REPCAP] = r;
        rc.nrep += 1; rc.steps += 1;
        rc.t = rc.t + c.dt;
        ds->nrep = rc.nrep; ds->steps = rc.steps; ds->t = rc.t;
      }
    }
    ds->tmax_ok[cur ^ 1] = 0;
    ds->slot[cur][0] = 0ull; ds->slot[cur][1] = 0ull; ds->slot[cur][2] = 0ull;
    rc.seq += 1;
    ds->seq = rc.seq;
  };

  for (int st = 0; st < nsteps; ++st) {
    stamp(st, 0);
    const int cur = (A.cur + st) & 1;
    const R* __restrict__ q = cur ? q1 : q0;
    R* __restrict__ qn = cur ? q0 : q1;
    bool stage_ok = true;
    if (ctl_warp) {
      if (lane == 0) {
        // this step's control first (the others need it at the next barrier),
        // then the previous step's record; a pending step is an applied one
        // (an error or a skip ends the loop), so t moves by its dt
        const double t_now = (rec && rc.have_pend) ? rc.t + rc.pend.dt : rc.t;
        const Ctl c0 = step_control_local(A, rc.msx, rc.msy, t_now, rc.err);
        s_ctl = c0;
        s_dtd[0] = (R)(c0.dt / A.dx);
        s_dtd[1] = (R)(c0.dt / A.dy);
        if (rec && rc.have_pend) { record(rc.pend, rc.pend_cur, 0); rc.have_pend = 0; }
      }
    } else {
      constexpr int NSTG = (HC + NTW - 1) / NTW;
      R qs[NSTG][NEQ], as[NSTG][NA1];
#pragma unroll
      for (int k = 0; k < NSTG; ++k) {
        const int idx = tid + k * NTW;
        if (idx < HC) {
          const int lx = idx % HW, ly = idx / HW;
          int gi = i0 - 2 + lx, gj = j0 - 2 + ly;
          if (!inner) { gi = map_i(gi, L); gj = map_j(gj, L); }
          WS_CHK(L, gi >= 0 && gi < L.nx && row_readable(gj, L), CHK_STAGE_READ);
          const R* src = q + row_off(gj, L) + gi;
#pragma unroll
          for (int c = 0; c < NEQ; ++c) qs[k][c] = __ldcg(src + c * L.pitch);
          if (NAUX > 0) {
            const R* asrc = aux + (long long)(gj + 2) * L.astride + gi;
#pragma unroll
            for (int c = 0; c < NAUX; ++c) as[k][c] = __ldcg(asrc + c * L.pitch);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < NSTG; ++k) {
        const int idx = tid + k * NTW;
        if (idx < HC) {
#pragma unroll
          for (int c = 0; c < NEQ; ++c) sQ[c * HC + idx] = qs[k][c];
#pragma unroll
          for (int c = 0; c < NAUX; ++c) sA[c * HC + idx] = as[k][c];
          R pc[NP1];
          if (NPR > 0) {
            prims_fast<S>(qs[k], as[k], P, pc);
#pragma unroll
            for (int c = 0; c < NPR; ++c) sP[c * HC + idx] = pc[c];
          }
          stage_ok = stage_ok && S::cell_ok(qs[k], as[k], pc, P);
        }
      }
    }
    const bool tile_clean = __syncthreads_and(stage_ok) != 0;
    stamp(st, 1);
    const Ctl ctl = s_ctl;
    if (ctl.skip) {
      if (rec) record(ctl, cur, 0);
      break;
    }
    const R dtdx = s_dtd[0], dtdy = s_dtd[1];
    unsigned long long key = ~0ull;
    // ---- x pass: warp r walks row r; lane l = x-edge i0-1+l
    if (!ctl_warp && warp < LW && j0 + warp < L.ny) {
      const int r = warp;
      const int cl = (r + 2) * HW + lane, cr = cl + 1;
      WS_CHK(L, cl >= 0 && cr < HC, CHK_EDGE_SMEM);
      const int ei = i0 - 1 + lane;
      R ap[NEQ], amn[NEQ], fl[NEQ], fr[NEQ];
      line_edge<S, R, ORDER, LIM, true, 1, HC>(sQ, sA, sP, P, L, cl, cr, ei, j0 + r,
                                               !tile_clean && lane >= 1 && lane <= 30 &&
                                                   ei <= L.nx,
                                               dtdx, key, ap, amn, fl, fr);
      if (cell_lane) {
        const int c = lane - 1;
#pragma unroll
        for (int m = 0; m < NEQ; ++m) {
          const R qc = sQ[m * HC + cr];
          R v = qc - dtdx * (ap[m] + amn[m]);
          if (ORDER == 2) v = v - dtdx * (fr[m] - fl[m]);
          WS_CHK(L, r * LW + c < LW * LW, CHK_X_SMEM);
          sX[m * (LW * LW) + r * LW + c] = v;
        }
      }
    }
    __syncthreads();
    stamp(st, 2);
    // ---- y pass: warp c walks column c; lane l = y-edge j0-1+l
    if (!ctl_warp && warp < LW && i0 + warp < L.nx) {
      const int c = warp;
      const int cl = lane * HW + c + 2, cr = cl + HW;
      WS_CHK(L, cl >= 0 && cr < HC, CHK_EDGE_SMEM);
      const int ej = j0 - 1 + lane;
      R ap[NEQ], amn[NEQ], fl[NEQ], fr[NEQ];
      line_edge<S, R, ORDER, LIM, true, 2, HC>(sQ, sA, sP, P, L, cl, cr, i0 + c, ej,
                                               !tile_clean && lane >= 1 && lane <= 30 &&
                                                   ej < L.ny_edges_y,
                                               dtdy, key, ap, amn, fl, fr);
      const int rr = lane - 1, o = rr * LW + c;
      WS_CHK(L, !cell_lane || (o >= 0 && o < LW * LW), CHK_X_SMEM);
      if (cell_lane) {
#pragma unroll
        for (int m = 0; m < NEQ; ++m) {
          R v = sX[m * (LW * LW) + o] - dtdy * (ap[m] + amn[m]);
          if (ORDER == 2) v = v - dtdy * (fr[m] - fl[m]);
          sX[m * (LW * LW) + o] = v;
        }
      }
    }
    __syncthreads();
    stamp(st, 3);
    // ---- row-coalesced store of the tile
    if (!ctl_warp) {
      for (int idx = tid; idx < LW * LW; idx += NTW) {
        const int rr = idx / LW, c = idx % LW;
        const int gi = i0 + c, gj = j0 + rr;
        if (gi < L.nx && gj < L.ny) {
          R* dst = qn + row_off(gj, L) + gi;
#pragma unroll
          for (int m = 0; m < NEQ; ++m) dst[m * L.pitch] = sX[m * (LW * LW) + idx];
          WS_CHK(L, gi >= 0 && gj >= 0, CHK_STORE);
          if (WS_CHECKED && L.chk) atomicAdd(&L.chk[1 + (long long)gj * L.nx + gi], 1u);
        }
      }
      if (key != ~0ull) atomicMax(&ds->slot[cur][2], NKEY_MAX - key);
    }
    const bool bad = __syncthreads_or(key != ~0ull) != 0;
    stamp(st, 4);
    // ---- grid barrier (see above)
    if (tid == 0) {
      red_add_release_gpu(&ds->mctr[cur], 1ull + (bad ? (1ull << 32) : 0ull));
      rc.uses[cur] += 1u;
      const unsigned need = rc.a0[cur] + rc.uses[cur] * nblk;
      unsigned long long w;
      long long spins = 0;
      int e = 0;
      while ((int)((unsigned)(w = ld_acquire_gpu(&ds->mctr[cur])) - need) < 0) {
        if (++spins > (1ll << 26)) { e = 2; break; }
      }
      s_err = e ? e : ((unsigned)(w >> 32) != rc.e0[cur] ? 1 : 0);
    }
    __syncthreads();
    stamp(st, 5);
    if (s_err) {
      if (rec) {
        if (s_err == 2) atomicCAS(&ds->err, 0, ERR_WAIT_TIMEOUT);
        else record(ctl, cur, 1);
      }
      break;
    }
    if (ctl_thr) {
      if (rec) { rc.pend = ctl; rc.pend_cur = cur; rc.have_pend = 1; }
      else rc.t = rc.t + ctl.dt;     // every CTA keeps t in step with the record
    }
  }
  if (rec && rc.have_pend) record(rc.pend, rc.pend_cur, 0);
}

// checked builds: NaN into every location no kernel may read -- the padding
// columns [nx, pitch) of each component row and the ghost rows of physical
// boundary sides (those are produced by index mapping, never loaded)
template <class R>
__global__ void k_canary(R* __restrict__ buf, const Layout L, int ncomp) {
  const long long per_row = (long long)ncomp * L.pitch;
  const long long n = (long long)(L.ny + 4) * per_row;
  const R nan = (R)NAN;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t / per_row) - 2;
    const int i = (int)((t % per_row) % L.pitch);
    const bool bc_row = (j < 0 && L.lo == ROWS_BC) || (j >= L.ny && L.hi == ROWS_BC);
    if (i >= L.nx || bc_row) buf[t] = nan;
  }
}

template <class S> struct LineGeom {
  static constexpr int LW = 29, HC = 33 * 33;
  template <class R> static constexpr size_t smem_bytes(bool persist = false,
                                                        bool fused = false) {
    return sizeof(R) * (size_t)((S::NEQ + S::NAUX + S::NPR) * HC +
                                (fused ? 2 : 1) * S::NEQ * LW * LW +
                                (persist ? (S::NEQ + S::NAUX) * HC : 0));
  }
};

// --------------------------------------------------------------------------
// layout conversion: host block (ncomp, nx+4, ny+4) F-order <-> SoA rows
template <class R, class HR>
__global__ void k_to_soa(const HR* __restrict__ hb, R* __restrict__ dst, int ncomp, int nx,
                         int ny, long long pitch) {
  // rows j in [-2, ny+2), columns i in [0, nx)
  const long long n = (long long)nx * (ny + 4);
  const int nxt = nx + 4;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % nx);
    const int jr = (int)(t / nx);  // j + 2
    const HR* s = hb + (long long)ncomp * ((i + 2) + (long long)nxt * jr);
    R* d = dst + (long long)jr * ncomp * pitch + i;
    for (int c = 0; c < ncomp; ++c) d[c * pitch] = (R)s[c];
  }
}

// full host block: interior from `cur`, ghost frame (x ghosts and BC rows)
// from `gsrc` via the same index mapping as fill_ghost; memory ghost rows
// from `gsrc`'s ghost rows.
template <class R, class HR>
__global__ void k_to_aos(const R* __restrict__ cur, const R* __restrict__ gsrc,
                         HR* __restrict__ hb, const Layout L, int ncomp) {
  const int nxt = L.nx + 4, nyt = L.ny + 4;
  const long long n = (long long)nxt * nyt;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const int ii = (int)(t % nxt), jj = (int)(t / nxt);
    const int i = ii - 2, j = jj - 2;
    const bool interior = (i >= 0 && i < L.nx && j >= 0 && j < L.ny);
    const R* base = interior ? cur : gsrc;
    int si = i, sj = j;
    if (!interior) {
      // x pass then y pass of grid.py:179-193 == q[map_x(i), map_y(j)]
      si = map_i(i, L);
      sj = (j < 0 || j >= L.ny) ? map_j(j, L) : j;
    }
    const R* s = base + row_off(sj, L) + si;
    HR* d = hb + (long long)ncomp * t;
    for (int c = 0; c < ncomp; ++c) d[c] = (HR)s[c * L.pitch];
  }
}

// acoustics-var: max over interior cells of c = aux[1] (static CFL speeds)
template <class R>
__global__ void k_static_speed(const R* __restrict__ aux, const Layout L, DevState* ds) {
  __shared__ unsigned long long sred[8];
  R m = (R)0;
  const long long n = (long long)L.nx * L.ny;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % L.nx), j = (int)(t / L.nx);
    R c = aux[(long long)(j + 2) * L.astride + L.pitch + i];
    // NaN propagates like numpy max (the positivity check reports it)
    m = (c != c || c > m) ? c : m;
  }
  unsigned long long b = block_max_u64<256>(Bits<R>::to(m), sred);
  if (threadIdx.x == 0) {
    atomicMax(&ds->static_bits[0], b);
    atomicMax(&ds->static_bits[1], b);
  }
}

// --------------------------------------------------------------------------
// batched pointwise plugin call (reference Kernel.solve)
template <class S, class R, int NI>
__global__ void k_riemann(const typename S::template Params<R> P, long long n,
                          const R* __restrict__ ql, const R* __restrict__ qr,
                          const R* __restrict__ al, const R* __restrict__ ar,
                          R* __restrict__ waves, R* __restrict__ speeds, R* __restrict__ amdq,
                          R* __restrict__ apdq, int* __restrict__ codes) {
  constexpr int NEQ = S::NEQ, NW = S::NW, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int NA1 = NAUX > 0 ? NAUX : 1, NP1 = NPR > 0 ? NPR : 1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    R a[NEQ], b[NEQ], xa[NA1], xb[NA1], pa[NP1], pb[NP1];
#pragma unroll
    for (int c = 0; c < NEQ; ++c) { a[c] = ql[c * n + e]; b[c] = qr[c * n + e]; }
#pragma unroll
    for (int c = 0; c < NAUX; ++c) { xa[c] = al[c * n + e]; xb[c] = ar[c * n + e]; }
    bool ok = true;
    if (NPR > 0) {
      S::template prims<IeeeMath>(a, xa, P, pa, ok);
      S::template prims<IeeeMath>(b, xb, P, pb, ok);
    }
    R sm;
    codes[e] = S::template probe<NI, IeeeMath>(a, b, pa, pb, xa, xb, P, sm, ok);
    R W[NW][NEQ], s[NW], am[NEQ], ap[NEQ];
    S::template solve<NI, IeeeMath>(a, b, pa, pb, xa, xb, P, W, s, am, ap, ok);
#pragma unroll
    for (int w = 0; w < NW; ++w) {
#pragma unroll
      for (int m = 0; m < NEQ; ++m) waves[(w * NEQ + m) * n + e] = W[w][m];
      speeds[w * n + e] = s[w];
    }
#pragma unroll
    for (int m = 0; m < NEQ; ++m) { amdq[m * n + e] = am[m]; apdq[m * n + e] = ap[m]; }
  }
}

// ghost fill of an F-order (ncomp, nx+4, ny+4) field: ghost (i, j) takes
// cell (map_x(i), map_y(j)) — the composition of grid.py's x then y pass
template <int UNUSED = 0>
__global__ void k_fill_ghost(double* __restrict__ d, int ncomp, int nx, int ny, int bcx, int bcy) {
  const int nxt = nx + 4, nyt = ny + 4;
  const long long n = (long long)nxt * nyt;
  Layout L{};
  L.nx = nx; L.ny = ny; L.bcx = bcx; L.bcy = bcy; L.lo = ROWS_BC; L.hi = ROWS_BC;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const int ii = (int)(t % nxt), jj = (int)(t / nxt);
    const int i = ii - 2, j = jj - 2;
    if (i >= 0 && i < nx && j >= 0 && j < ny) continue;
    const int si = map_i(i, L) + 2, sj = map_j(j, L) + 2;
    const double* s = d + (long long)ncomp * (si + (long long)nxt * sj);
    double* o = d + (long long)ncomp * t;
    for (int c = 0; c < ncomp; ++c) o[c] = s[c];
  }
}

}  // namespace ws
