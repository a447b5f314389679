// ws_kernels.cuh — the step kernels.
//
//   k_speeds  : CFL pre-pass.  Every reference edge (x: i in [0,nx], j in
//               [0,ny); y: i in [0,nx), j in [0,ny], sweep.py:111-163, 250)
//               is probed: admissibility in the reference order and max |s|,
//               reduced warp-shuffle -> block -> one atomicMax per CTA.
//   k_update  : fused edge + update kernel.  One CTA owns a TX x TY tile; the
//               tile plus an H-cell halo is staged in shared memory once,
//               per-cell primitives are computed once per cell, every edge
//               is solved once per tile, waves are limited against their
//               upwind neighbour, and the donor-cell update (reference order,
//               sweep.py:275-277) plus the correction flux are applied in
//               registers.  No fluctuation arrays ever reach HBM.  The last
//               CTA to finish commits the step (report, t, counters).
//   k_to_soa / k_to_aos / k_static_speed : layout conversion, acoustics setup.
#pragma once
#include <type_traits>

#include "ws_solvers.cuh"

namespace ws {

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

// --------------------------------------------------------------------------
// CFL / admissibility pre-pass
template <class S, class R, int TX, int TY>
__global__ void __launch_bounds__(TX * TY)
k_speeds(const R* __restrict__ q, const R* __restrict__ aux, const Layout L,
         const typename S::template Params<R> P, const int cur, DevState* __restrict__ ds) {
  constexpr int NT = TX * TY, NEQ = S::NEQ, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int HX = TX + 1, HY = TY + 1, HC = HX * HY;
  __shared__ R sQ[NEQ][HC];
  __shared__ R sA[NAUX > 0 ? NAUX : 1][HC];
  __shared__ R sP[NPR > 0 ? NPR : 1][HC];
  __shared__ unsigned long long sred[NT / 32];
  {
    volatile const DevState* vds = ds;
    if (vds->err || vds->finished) return;   // stable for the whole kernel
  }
  const int tid = threadIdx.x;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  // tile cell (lx, ly) = cell (i0 - 1 + lx, j0 - 1 + ly)
  for (int idx = tid; idx < HC; idx += NT) {
    int lx = idx % HX, ly = idx / HX;
    int gi = map_i(i0 - 1 + lx, L), gj = map_j(j0 - 1 + ly, L);
    R qc[NEQ], ac[NAUX > 0 ? NAUX : 1], pc[NPR > 0 ? NPR : 1];
    const R* src = q + row_off(gj, L) + gi;
#pragma unroll
    for (int c = 0; c < NEQ; ++c) { qc[c] = src[c * L.pitch]; sQ[c][idx] = qc[c]; }
    if (NAUX > 0) {
      const R* asrc = aux + (long long)(gj + 2) * L.astride + gi;
#pragma unroll
      for (int c = 0; c < NAUX; ++c) { ac[c] = asrc[c * L.pitch]; sA[c][idx] = ac[c]; }
    }
    if (NPR > 0) {
      S::prims(qc, ac, P, pc);
#pragma unroll
      for (int c = 0; c < NPR; ++c) sP[c][idx] = pc[c];
    }
  }
  __syncthreads();

  const int li = tid % TX, lj = tid / TX;
  const int i = i0 + li, j = j0 + lj;
  R mx = (R)0, my = (R)0;
  unsigned long long key = ~0ull;
  auto edge = [&](auto ni_tag, int cl, int cr, int dir, int ei, int ej) {
    constexpr int NI = decltype(ni_tag)::value;
    R ql[NEQ], qr[NEQ], al[NAUX > 0 ? NAUX : 1], ar[NAUX > 0 ? NAUX : 1];
    R pl[NPR > 0 ? NPR : 1], pr[NPR > 0 ? NPR : 1];
#pragma unroll
    for (int c = 0; c < NEQ; ++c) { ql[c] = sQ[c][cl]; qr[c] = sQ[c][cr]; }
#pragma unroll
    for (int c = 0; c < NAUX; ++c) { al[c] = sA[c][cl]; ar[c] = sA[c][cr]; }
#pragma unroll
    for (int c = 0; c < NPR; ++c) { pl[c] = sP[c][cl]; pr[c] = sP[c][cr]; }
    R sm;
    int code = S::template probe<NI>(ql, qr, pl, pr, al, ar, P, sm);
    if (code) {
      unsigned long long k = err_key(dir, ei, L.j_off + ej, (code & 0xff) - 1, code >> 8, L.nx);
      key = k < key ? k : key;
    }
    return sm;
  };
  using NX = std::integral_constant<int, 1>;
  using NY = std::integral_constant<int, 2>;
  if (i <= L.nx && j < L.ny) {
    R s = edge(NX{}, (lj + 1) * HX + li, (lj + 1) * HX + li + 1, 0, i, j);
    mx = nmax(mx, s);   // NaN-free unless inadmissible (flagged)
  }
  if (i < L.nx && j < L.ny_edges_y) {
    R s = edge(NY{}, lj * HX + li + 1, (lj + 1) * HX + li + 1, 1, i, j);
    my = nmax(my, s);
  }
  if (key != ~0ull) atomicMax(&ds->slot[cur][2], ~key);
  unsigned long long bx = block_max_u64<NT>(Bits<R>::to(mx), sred);
  __syncthreads();
  unsigned long long by = block_max_u64<NT>(Bits<R>::to(my), sred);
  if (tid == 0) {
    atomicMax(&ds->slot[cur][0], bx);
    atomicMax(&ds->slot[cur][1], by);
  }
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
      v->err = ERR_KERNEL; v->err_key = ~nkey; v->err_step = v->steps;
    } else if (c.stationary) {
      v->err = ERR_STATIONARY; v->err_step = v->steps;
    } else {
      long long n = v->nrep;
      Report r;
      r.dt = c.dt;
      r.cfl = c.dt * (c.msx / A.dx + c.msy / A.dy);   // driver.py:501
      r.msx = c.msx; r.msy = c.msy;
      ds->rep[n % REPCAP] = r;
      v->nrep = n + 1;
      v->steps = v->steps + 1;
      v->t = v->t + c.dt;
    }
  }
  // the next step's speeds kernel accumulates into the other slot
  v->slot[A.cur ^ 1][0] = 0ull; v->slot[A.cur ^ 1][1] = 0ull; v->slot[A.cur ^ 1][2] = 0ull;
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
  template <class R> static constexpr size_t smem_bytes() {
    return sizeof(R) * (size_t)((NEQ + NAUX + NPR) * HC + EBUF);
  }
};

template <class S, class R, int ORDER, int LIM, int TX, int TY, int NT, bool CHECKS>
__global__ void __launch_bounds__(NT)
k_update(const R* __restrict__ q, const R* __restrict__ aux, R* __restrict__ qn, const Layout L,
         const typename S::template Params<R> P, const StepArgs A, DevState* __restrict__ ds) {
  using G = TileGeom<S, ORDER, TX, TY>;
  constexpr int NEQ = S::NEQ, NW = S::NW, NAUX = S::NAUX, NPR = S::NPR;
  constexpr int H = G::H, HX = G::HX, HC = G::HC;
  constexpr int NEXC = G::NEXC, NEX = G::NEX, NEY = G::NEY, NEST = G::NEST, NIST = G::NIST;
  constexpr int KEX = (NEX + NT - 1) / NT, KEY = (NEY + NT - 1) / NT;
  constexpr int KC = (TX * TY) / NT;
  constexpr int NA1 = NAUX > 0 ? NAUX : 1, NP1 = NPR > 0 ? NPR : 1;
  static_assert(KC * NT == TX * TY, "tile must be a multiple of the block");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sQ = reinterpret_cast<R*>(smem_raw);
  R* sA = sQ + NEQ * HC;
  R* sP = sA + NAUX * HC;
  R* sE = sP + NPR * HC;   // wave records (order 2), then fluctuation/flux records
  __shared__ Ctl s_ctl;

  const int tid = threadIdx.x;
  if (tid == 0) s_ctl = step_control<R>(A, ds, !CHECKS);
  __syncthreads();
  const Ctl ctl = s_ctl;

  if (!ctl.skip) {
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
    const R dtdx = (R)(ctl.dt / A.dx);
    const R dtdy = (R)(ctl.dt / A.dy);
    unsigned long long key = ~0ull;

    // ---- stage the tile + halo (BC by index mapping) and per-cell primitives
    for (int idx = tid; idx < HC; idx += NT) {
      int lx = idx % HX, ly = idx / HX;
      int gi = map_i(i0 - H + lx, L), gj = map_j(j0 - H + ly, L);
      R qc[NEQ], ac[NA1], pc[NP1];
      const R* src = q + row_off(gj, L) + gi;
#pragma unroll
      for (int c = 0; c < NEQ; ++c) { qc[c] = src[c * L.pitch]; sQ[c * HC + idx] = qc[c]; }
      if (NAUX > 0) {
        const R* asrc = aux + (long long)(gj + 2) * L.astride + gi;
#pragma unroll
        for (int c = 0; c < NAUX; ++c) { ac[c] = asrc[c * L.pitch]; sA[c * HC + idx] = ac[c]; }
      }
      if (NPR > 0) {
        S::prims(qc, ac, P, pc);
#pragma unroll
        for (int c = 0; c < NPR; ++c) sP[c * HC + idx] = pc[c];
      }
    }
    __syncthreads();

    R q1[KC][NEQ], dfx[KC][NEQ];

    // one sweep direction: solve -> (limit) -> fluctuation/flux records in sE
    auto sweep = [&](auto ni_tag) {
      constexpr int NI = decltype(ni_tag)::value;
      constexpr int NE = (NI == 1) ? NEX : NEY;
      constexpr int KE = (NI == 1) ? KEX : KEY;
      R fm[KE][NEQ], fp[KE][NEQ], ff[KE][NEQ];
      // solve every edge of the tile (+ the limiter's neighbours for order 2)
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
          S::template solve<NI>(ql, qr, pl, pr, al, ar, P, W, s, fm[k], fp[k]);
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
              int code = S::template probe<NI>(ql, qr, pl, pr, al, ar, P, sm);
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
              R th = (dow != (R)0) ? dup / dow : (R)0;
              R ph = limiter_phi<LIM>(th);
              R a = fabs(so);
              R coef = a * ((R)1 - dtdn * a);
#pragma unroll
              for (int m = 0; m < NEQ; ++m) {
                R wl = ph * own[m];
                f[m] = (w == 0) ? coef * wl : f[m] + coef * wl;
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
      const int li = cidx % TX, lr = cidx / TX;
      const int el = lr * (TX + 1) + li, er = el + 1;
#pragma unroll
      for (int m = 0; m < NEQ; ++m) {
        R qc = sQ[m * HC + (lr + H) * HX + li + H];
        q1[kc][m] = qc - dtdx * (sE[(NEQ + m) * NIST + el] + sE[m * NIST + er]);
        if (ORDER == 2) dfx[kc][m] = sE[(2 * NEQ + m) * NIST + er] - sE[(2 * NEQ + m) * NIST + el];
      }
    }
    __syncthreads();

    // ---- y sweep, the y term, then the correction fluxes
    sweep(NY{});
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      const int cidx = tid + kc * NT;
      const int li = cidx % TX, lr = cidx / TX;
      const int el = lr * TX + li, eu = el + TX;
      const int gi = i0 + li, gj = j0 + lr;
      R out[NEQ];
#pragma unroll
      for (int m = 0; m < NEQ; ++m) {
        R v = q1[kc][m] - dtdy * (sE[(NEQ + m) * NIST + el] + sE[m * NIST + eu]);
        if (ORDER == 2) {
          v = v - dtdx * dfx[kc][m];
          v = v - dtdy * (sE[(2 * NEQ + m) * NIST + eu] - sE[(2 * NEQ + m) * NIST + el]);
        }
        out[m] = v;
      }
      if (gi < L.nx && gj < L.ny) {
        R* dst = qn + row_off(gj, L) + gi;
#pragma unroll
        for (int m = 0; m < NEQ; ++m) dst[m * L.pitch] = out[m];
      }
    }
    if (CHECKS && key != ~0ull) atomicMax(&ds->slot[A.cur][2], ~key);
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
    if (NPR > 0) { S::prims(a, xa, P, pa); S::prims(b, xb, P, pb); }
    R sm;
    codes[e] = S::template probe<NI>(a, b, pa, pb, xa, xb, P, sm);
    R W[NW][NEQ], s[NW], am[NEQ], ap[NEQ];
    S::template solve<NI>(a, b, pa, pb, xa, xb, P, W, s, am, ap);
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
