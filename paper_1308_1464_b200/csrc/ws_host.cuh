// ws_host.cuh — host-side launch machinery shared by the C-ABI translation
// unit (wavestep.cu) and the per-solver instantiation units (ws_inst_*.cu).
#pragma once
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "../../include/wavestep.h"
#include "ws_kernels.cuh"

using namespace ws;

struct ws_handle;

namespace wsh {

template <class S, class R, int ORDER> struct TileCfg {
  static constexpr int TX = 32, TY = 16, NT = 256;
};
// Euler-Roe's 15-value wave record would cap residency at 1 CTA/SM at 32x16
template <class R> struct TileCfg<EulerRoe, R, 2> {
  static constexpr int TX = 32, TY = 8, NT = 256;
};
constexpr int SPD_TX = 32, SPD_NT = 256;
// pre-pass tile height: 32 rows (4 cells per thread) when the staged halo tile
// fits the 48 KB static shared-memory window, else 16
template <class S, class R> constexpr int spd_ty() {
  return (S::NEQ + S::NAUX + S::NPR) * 33 * 33 * sizeof(R) <= 46 * 1024 ? 32 : 16;
}

struct Ops {
  void (*speeds)(ws_handle*, const void* q, int cur, int part, cudaStream_t);
  void (*update)(ws_handle*, const void* q, void* qn, const StepArgs&, cudaStream_t);
  void (*to_soa)(ws_handle*, const void* stage, void* dst, int ncomp, cudaStream_t);
  void (*to_aos)(ws_handle*, const void* cur, const void* gsrc, void* stage, cudaStream_t);
  void (*to_aos_aux)(ws_handle*, void* stage, cudaStream_t);   // aux + BC ghost frame
  void (*canary)(ws_handle*, cudaStream_t);   // checked builds: NaN where nothing may read
  int (*update_ctas)(ws_handle*, const StepArgs&);   // CTAs of a shard step part
  void (*static_speed)(ws_handle*, cudaStream_t);
  void (*prepare)();   // one-time kernel attributes (never inside a capture)
  // ws_run on a small static-speed grid: all steps in one cooperative launch
  // (k_run_small); returns 0 when it does not apply (nothing launched)
  int (*run_small)(ws_handle*, const StepArgs&, int nsteps, cudaStream_t);
  int static_speeds;   // solver has q-independent speeds
  int can_fuse_line;   // warp-line kernel has the fused next-step CFL epilogue
  int tile_prepass;    // solver has tile accumulators (S::HAS_TILE)
  int nacc;            // ints per tile of those accumulators
};

}  // namespace wsh

struct ws_handle {
  using Ops = wsh::Ops;
  ws_desc d{};
  int neq = 0, naux = 0;
  size_t esz = 8;
  Layout L{};
  void* q[2] = {nullptr, nullptr};
  void* aux = nullptr;
  DevState* ds = nullptr;
  bool own_q[2] = {false, false}, own_aux = false, own_ds = false;
  void* stage[2] = {nullptr, nullptr};   // upload staging (host layout), alternating
  size_t stage_bytes[2] = {0, 0};
  int up_idx = 0;                        // staging buffer of the next upload
  void* stage_out = nullptr;     // download staging: a download and the next upload overlap
  size_t stage_out_bytes = 0;
  unsigned* chk = nullptr;       // checked builds: {violation bits, per-cell write counts}
  void* stage_aux = nullptr;     // aux in the host layout with its BC ghost frame
  size_t stage_aux_bytes = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t cstream = nullptr;  // upload H2D copies (staging only)
  cudaStream_t last_stream = nullptr;
  cudaEvent_t ev_order = nullptr;  // issue-order hand-off between streams (pick)
  bool order_recorded = false;     // ev_order already marks the last ordering point
  cudaEvent_t ev_in[2] = {nullptr, nullptr};    // staging b consumed (its next H2D may start)
  cudaEvent_t ev_copy[2] = {nullptr, nullptr};  // staging b filled by its H2D
  cudaEvent_t ev_out = nullptr;    // download staging copied out (next download may refill it)
  long long enq = 0;            // steps enqueued since upload (== committed after a poll)
  long long nrep_seen = 0;
  // a t_final control was enqueued since the last resync: the device may have
  // stopped early, so enq can run ahead of the committed steps (and of the
  // buffer parity).  The next call with another control resyncs first.
  bool tf_pending = false;
  double tf_value = 0.0;
  bool multi = false;           // row-strip shard with memory ghost rows
  bool uploaded = false;
  double host_static[2] = {0, 0};
  Ops ops{};
  std::vector<char> params;     // typed Params<R> blob
  // graph cache
  cudaGraphExec_t gexec = nullptr;
  ws_ctl gctl{};
  cudaStream_t gstream = nullptr;
  long long launches = 0;
  long long graph_launches = 0;  // kernels per replay of the 2-step graph
  // ws_capture_begin / _end: the counts before a caller-side capture
  bool cap_open = false;
  long long cap_enq = 0, cap_launches = 0;
  bool run_small = true;        // ws_run: multi-step k_run_small where it applies
  bool fused = false;           // next-step CFL maxima computed in the update epilogue
  bool need_prepass = true;     // fused mode: slot of the current state not yet filled
  int* borders = nullptr;       // tile-border counters of the fused epilogue
  unsigned long long* trace = nullptr;   // CTA timeline buffer (WS_TRACE=1)
  bool line_kernel = true;      // warp-per-line k_update_w (else the smem-tile k_update)
  bool speeds_smem = false;     // shared-memory tile pre-pass (else the register k_speeds_w)
  bool speeds_exact = false;    // probe every edge (k_speeds_w) even where a filter exists
  bool speeds_edge = false;     // per-edge candidate filter (k_speeds_b) instead of whole tiles
  bool tile_prepass = false;    // k_speeds_t, fed by the update's per-tile bound maxima
  void* tmax = nullptr;         // [2][ntiles][4] R per-tile bound maxima
  bool pdl = true;              // programmatic dependent launch of the step kernels
  bool persist = true;          // persistent prefetching line kernel where it applies
  cudaError_t launch_err = cudaSuccess;  // first failed cudaLaunchKernelEx (reported once)
  void* peers_dev = nullptr;    // device table of the shards' DevState (device-side reduce)
  size_t border_bytes = 0;
  std::string err;
};

namespace wsh {

// defined in wavestep.cu (per-handle message, or the thread's create error)
int fail(ws_handle* h, int code, const std::string& msg);

inline int cuda_fail(ws_handle* h, cudaError_t e, const char* where) {
  std::string m = std::string(where) + ": " + cudaGetErrorString(e);
  return fail(h, WS_ERR_CUDA, m);
}

#define WS_CUDA(h, call)                                   \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return cuda_fail((h), e_, #call); \
  } while (0)

// launch status of everything enqueued since the last check: a failed
// cudaLaunchKernelEx (returned, not necessarily sticky) or the runtime's last error
inline cudaError_t launch_status(ws_handle* h) {
  cudaError_t e = h->launch_err;
  h->launch_err = cudaSuccess;
  const cudaError_t l = cudaGetLastError();
  return e != cudaSuccess ? e : l;
}

// Stream of an ABI call (null: the handle's own stream).  Operations on one
// handle run in issue order whatever streams they are issued on: switching
// streams makes the new stream wait for everything issued before.
inline cudaStream_t pick(ws_handle* h, void* s) {
  cudaStream_t st = s ? reinterpret_cast<cudaStream_t>(s) : h->stream;
  if (h->last_stream && h->last_stream != st && h->ev_order) {
    if (!h->order_recorded) cudaEventRecord(h->ev_order, h->last_stream);
    cudaStreamWaitEvent(st, h->ev_order, 0);
  }
  h->order_recorded = false;
  h->last_stream = st;
  return st;
}

// persistent grid: resident CTAs (occupancy query, cached per kernel), capped
// by the tile count
template <class K>
int persistent_grid(K kernel, int nt, size_t smem, int nx, int ny, int tx, int ty) {
  static std::unordered_map<const void*, int> cache;   // resident CTAs per SM, per kernel
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  auto it = cache.find((const void*)kernel);
  int per_sm;
  if (it == cache.end()) {
    per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, nt, smem);
    if (per_sm < 1) per_sm = 1;
    cache[(const void*)kernel] = per_sm;
  } else {
    per_sm = it->second;
  }
  const long long tiles = (long long)((nx + tx - 1) / tx) * ((ny + ty - 1) / ty);
  const long long g = (long long)per_sm * sms;
  return (int)(tiles < g ? tiles : g);
}

// kernel launch, with programmatic dependent launch when enabled (the two
// per-step kernels: k_speeds_w and k_update_w, see ws_common.cuh pdl_*)
template <class... KArgs, class... Args>
inline void launch(ws_handle* h, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                   cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = h->pdl ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k, args...);
  if (e != cudaSuccess && h->launch_err == cudaSuccess) h->launch_err = e;
}

// ---- typed launchers -----------------------------------------------------
template <class S, class R, int ORDER, int LIM> struct Impl {
  using P = typename S::template Params<R>;
  using C = TileCfg<S, R, ORDER>;
  using G = TileGeom<S, ORDER, C::TX, C::TY>;

  static const P& prm(ws_handle* h) { return *reinterpret_cast<const P*>(h->params.data()); }

  static void speeds(ws_handle* h, const void* q, int cur, int part, cudaStream_t st) {
    if (h->speeds_smem && part == 0 && h->L.npeers == 0 && h->L.hsides == 0) {
      constexpr int TY = spd_ty<S, R>();
      dim3 grid((h->L.nx + 1 + SPD_TX - 1) / SPD_TX, (h->L.ny + 1 + TY - 1) / TY);
      k_speeds<S, R, SPD_TX, TY, SPD_NT><<<grid, SPD_NT, 0, st>>>(
          static_cast<const R*>(q), static_cast<const R*>(h->aux), h->L, prm(h), cur, h->ds);
    } else if (HasTile<S>::value && h->tile_prepass) {
      // a row-strip shard's split pre-pass: part 1 (overlapping the halo
      // exchange) is empty, part 2 (after it) probes every candidate tile
      if (part == 1) return;
      if constexpr (HasTile<S>::value) {
        constexpr int LW = 29, NWT = 8;
        const int nt = ((h->L.nx + LW - 1) / LW) * ((h->L.ny + LW - 1) / LW);
        // decisions interleaved over the CTAs, at most TILE_LIST tiles each
        long long ctas = 148 * 4;
        if ((long long)nt > ctas * TILE_LIST) ctas = ((long long)nt + TILE_LIST - 1) / TILE_LIST;
        // split each tile's rows over up to 4 CTAs while the decisions still
        // take one pass of the grid's threads
        int spl = (int)((ctas * NWT * 32) / nt);
        spl = spl < 1 ? 1 : (spl > 4 ? 4 : spl);
        if (ctas > (long long)nt * spl) ctas = (long long)nt * spl;
        launch(h, k_speeds_t<S, R, NWT>, dim3((unsigned)ctas), dim3(NWT * 32), 0, st,
               static_cast<const R*>(q), static_cast<const R*>(h->aux),
               static_cast<const int4*>(h->tmax), h->L, prm(h), cur, spl,
               h->ds);
      }
    } else if (HasBound<S>::value && !h->speeds_exact) {
      // candidate-filter pre-pass (exact result, see k_speeds_b)
      if constexpr (HasBound<S>::value) {
        constexpr int KC = 8, NW = 4, MB = S::NEQ <= 3 ? 8 : 4;
        dim3 grid((h->L.nx + 1 + 30) / 31,
                  part == 2 ? 2 : (h->L.ny + 1 + KC * NW - 1) / (KC * NW));
        launch(h, k_speeds_b<S, R, KC, NW, MB, 6>, grid, dim3(NW * 32), 0, st,
               static_cast<const R*>(q), static_cast<const R*>(h->aux), h->L, prm(h), cur, part,
               h->ds);
      }
    } else {
      // register pre-pass: 8 edge rows per warp, 4 warps per CTA (the best of
      // the geometries measured in round 1, DESIGN.md perf log)
      constexpr int KC = 8, NW = 4, MB = S::NEQ <= 3 ? 8 : 4;
      dim3 grid((h->L.nx + 1 + 30) / 31,
                part == 2 ? 2 : (h->L.ny + 1 + KC * NW - 1) / (KC * NW));
      launch(h, k_speeds_w<S, R, KC, NW, 1, MB>, grid, dim3(NW * 32), 0, st,
             static_cast<const R*>(q), static_cast<const R*>(h->aux), h->L, prm(h), cur, part,
             h->ds);
    }
    h->launches++;
  }

  template <bool CHECKS, bool FUSED> static auto kern() {
    return k_update<S, R, ORDER, LIM, C::TX, C::TY, C::NT, CHECKS, FUSED>;
  }

  static void prepare() {
    if constexpr (S::STATIC_SPEEDS)
      cudaFuncSetAttribute(k_run_small<S, R, ORDER, LIM, NWR>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)small_smem());
    const int lsmem = (int)LineGeom<S>::template smem_bytes<R>();
    cudaFuncSetAttribute(kern_w<true, false>(), cudaFuncAttributeMaxDynamicSharedMemorySize, lsmem);
    cudaFuncSetAttribute(kern_w<false, false>(), cudaFuncAttributeMaxDynamicSharedMemorySize, lsmem);
    if constexpr (PERSIST_W) {
      const int psmem = (int)LineGeom<S>::template smem_bytes<R>(true);
      cudaFuncSetAttribute(kern_w<true, false, true>(), cudaFuncAttributeMaxDynamicSharedMemorySize, psmem);
      cudaFuncSetAttribute(kern_w<false, false, true>(), cudaFuncAttributeMaxDynamicSharedMemorySize, psmem);
    }
    if constexpr (CAN_FUSE)
      cudaFuncSetAttribute(kern_w<false, true>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)LineGeom<S>::template smem_bytes<R>(false, true));
    const int smem = (int)G::template smem_bytes<R>();
    cudaFuncSetAttribute(kern<true, false>(), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern<false, false>(), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern<false, true>(), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  }

  template <bool CHECKS, bool FUSED> static void update_t(ws_handle* h, const void* q, void* qn,
                                                          const StepArgs& a, cudaStream_t st) {
    auto k = kern<CHECKS, FUSED>();
    const size_t smem = G::template smem_bytes<R>();
    dim3 grid(persistent_grid(k, C::NT, smem, h->L.nx, h->L.ny, C::TX, C::TY));
    k<<<grid, C::NT, smem, st>>>(static_cast<const R*>(q), static_cast<const R*>(h->aux),
                                 static_cast<R*>(qn), h->L, prm(h), a, h->ds);
    h->launches++;
  }

  // warps per CTA of the warp-line kernel: 29 lines / 10 ~ 97 % at 2 CTAs/SM;
  // 4-component systems stage 141 KB (fp64) -> 1 CTA/SM of 15 warps (97 %)
  static constexpr int LNW = (S::NEQ >= 4 && sizeof(R) == 8 && !WS_GAS2) ? 15
                             : (S::NEQ <= 3 && sizeof(R) == 8) ? WS_LNW3 : 10;
  static constexpr bool CAN_FUSE = !S::STATIC_SPEEDS && S::NAUX == 0 && S::NPR <= S::NEQ;
  // persistent form: one CTA of 15 warps per SM (29 lines / 15 ~ 97 %)
  static constexpr int LNWP = 15;
  template <bool CHECKS, bool FUSED, bool PERSIST = false> static auto kern_w() {
    return k_update_w<S, R, ORDER, LIM, PERSIST ? LNWP : LNW, CHECKS, FUSED, PERSIST>;
  }
  // one CTA per SM (4-component fp64): persistent CTAs prefetch the next tile
  static constexpr bool PERSIST_W = S::NEQ >= 4 && sizeof(R) == 8 && !WS_GAS2;

  // tile rows of a step part (StepArgs::part; 0 = the whole step)
  static int part_rows(const ws_handle* h, const StepArgs& a) {
    const int nty = (h->L.ny + 28) / 29;
    return a.part == 0 ? nty : a.part == 1 ? a.tr_lo + nty - a.tr_hi : a.tr_hi - a.tr_lo;
  }
  // CTAs the line kernel launches for a part of a shard's step (no checks,
  // no fused epilogue: the shard form)
  static int update_ctas(ws_handle* h, const StepArgs& a) {
    const int rows = part_rows(h, a);
    if (rows <= 0) return 0;
    if constexpr (PERSIST_W) {
      if (h->persist)
        return persistent_grid(kern_w<false, false, true>(), LNWP * 32,
                               LineGeom<S>::template smem_bytes<R>(true), h->L.nx, rows * 29,
                               29, 29);
    }
    return ((h->L.nx + 28) / 29) * rows;
  }

  template <bool CHECKS, bool FUSED> static void update_w(ws_handle* h, const void* q, void* qn,
                                                          const StepArgs& a, cudaStream_t st) {
    const int rows = part_rows(h, a);
    if (rows <= 0) return;    // an empty part (a strip of one or two tile rows)
    if constexpr (PERSIST_W && !FUSED) {
      if (h->persist) {
        auto k = kern_w<CHECKS, false, true>();
        const size_t smem = LineGeom<S>::template smem_bytes<R>(true);
        dim3 grid(persistent_grid(k, LNWP * 32, smem, h->L.nx, rows * 29, 29, 29));
        launch(h, k, grid, dim3(LNWP * 32), smem, st, static_cast<const R*>(q),
               static_cast<const R*>(h->aux), static_cast<R*>(qn), h->L, prm(h), a, h->ds);
        h->launches++;
        return;
      }
    }
    auto k = kern_w<CHECKS, FUSED>();
    const size_t smem = LineGeom<S>::template smem_bytes<R>(false, FUSED);
    dim3 grid((h->L.nx + 28) / 29, rows);
    launch(h, k, grid, dim3(LNW * 32), smem, st, static_cast<const R*>(q),
           static_cast<const R*>(h->aux), static_cast<R*>(qn), h->L, prm(h), a, h->ds);
    h->launches++;
    if (FUSED) {
      // tile-border edges of the new state, into the next step's slot
      k_border<S, R, 29, 256><<<148 * 2, 256, 0, st>>>(static_cast<const R*>(qn), h->L, prm(h),
                                                       a.cur ^ 1, h->ds);
      h->launches++;
    }
  }

  static void update(ws_handle* h, const void* q, void* qn, const StepArgs& a, cudaStream_t st) {
    if (h->line_kernel) {
      if (S::STATIC_SPEEDS && !h->multi) update_w<true, false>(h, q, qn, a, st);
      else if constexpr (CAN_FUSE) {
        if (h->fused) update_w<false, true>(h, q, qn, a, st);
        else update_w<false, false>(h, q, qn, a, st);
      } else {
        update_w<false, false>(h, q, qn, a, st);
      }
      return;
    }
    if (S::STATIC_SPEEDS && !h->multi) update_t<true, false>(h, q, qn, a, st);
    else if (h->fused) update_t<false, true>(h, q, qn, a, st);
    else update_t<false, false>(h, q, qn, a, st);
  }

  static void to_soa(ws_handle* h, const void* stage, void* dst, int ncomp, cudaStream_t st) {
    int blocks = 148 * 8;
    k_to_soa<R, R><<<blocks, 256, 0, st>>>(static_cast<const R*>(stage), static_cast<R*>(dst),
                                           ncomp, h->L.nx, h->L.ny, h->L.pitch);
    h->launches++;
  }

  static void to_aos(ws_handle* h, const void* cur, const void* gsrc, void* stage,
                     cudaStream_t st) {
    int blocks = 148 * 8;
    k_to_aos<R, R><<<blocks, 256, 0, st>>>(static_cast<const R*>(cur),
                                           static_cast<const R*>(gsrc), static_cast<R*>(stage),
                                           h->L, h->neq);
    h->launches++;
  }

  static void to_aos_aux(ws_handle* h, void* stage, cudaStream_t st) {
    Layout La = h->L;
    La.rstride = h->L.astride;     // aux rows: naux component rows per j
    const R* a = static_cast<const R*>(h->aux);
    k_to_aos<R, R><<<148 * 8, 256, 0, st>>>(a, a, static_cast<R*>(stage), La, h->naux);
    h->launches++;
  }

  static void canary(ws_handle* h, cudaStream_t st) {
    for (int b = 0; b < 2; ++b) {
      k_canary<R><<<148 * 4, 256, 0, st>>>(static_cast<R*>(h->q[b]), h->L, h->neq);
      h->launches++;
    }
    if (h->naux > 0) {
      k_canary<R><<<148 * 4, 256, 0, st>>>(static_cast<R*>(h->aux), h->L, h->naux);
      h->launches++;
    }
  }

  static void static_speed(ws_handle* h, cudaStream_t st) {
    if (S::NAUX > 0) {
      k_static_speed<R><<<148 * 4, 256, 0, st>>>(static_cast<const R*>(h->aux), h->L, h->ds);
      h->launches++;
    }
  }

  // k_run_small: one 30-warp CTA per tile, every tile resident at once
  static constexpr int NWR = 30;
  static constexpr size_t small_smem() {
    return sizeof(R) * (size_t)((S::NEQ + S::NAUX + S::NPR) * 33 * 33 + S::NEQ * 29 * 29);
  }
  static int run_small(ws_handle* h, const StepArgs& a, int nsteps, cudaStream_t st) {
    if constexpr (!S::STATIC_SPEEDS) {
      return 0;
    } else {
      if (h->multi || !h->line_kernel || !h->run_small || (h->trace && !WS_RS_PROF)) return 0;
      auto k = k_run_small<S, R, ORDER, LIM, NWR>;
      static int per_sm = -1, sms = 0;
      if (per_sm < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NWR * 32, small_smem()) !=
            cudaSuccess) {
          cudaGetLastError();
          per_sm = 0;
        }
      }
      const long long ntiles = (long long)((h->L.nx + 28) / 29) * ((h->L.ny + 28) / 29);
      if (per_sm < 1 || ntiles > (long long)per_sm * sms) return 0;
      // inside a caller's stream capture: the per-step kernels (a refused
      // cooperative launch would invalidate the capture)
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return 0;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)ntiles);
      cfg.blockDim = dim3(NWR * 32);
      cfg.dynamicSmemBytes = small_smem();
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;   // co-residency of every CTA
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const cudaError_t e = cudaLaunchKernelEx(&cfg, k, static_cast<R*>(h->q[0]),
                                               static_cast<R*>(h->q[1]),
                                               static_cast<const R*>(h->aux), h->L, prm(h), a,
                                               nsteps, h->ds);
      if (e != cudaSuccess) {
        // refused (e.g. the co-resident grid does not fit beside other work
        // on the device): nothing was enqueued, the caller takes the
        // per-step path
        cudaGetLastError();
        return 0;
      }
      h->launches++;
      return 1;
    }
  }

  static Ops ops() {
    Ops o;
    o.run_small = &run_small;
    o.speeds = &speeds;
    o.update = &update;
    o.to_soa = &to_soa;
    o.to_aos = &to_aos;
    o.to_aos_aux = &to_aos_aux;
    o.canary = &canary;
    o.update_ctas = &update_ctas;
    o.static_speed = &static_speed;
    o.prepare = &prepare;
    o.static_speeds = S::STATIC_SPEEDS ? 1 : 0;
    o.can_fuse_line = CAN_FUSE ? 1 : 0;
    o.tile_prepass = HasTile<S>::value ? 1 : 0;
    o.nacc = NAcc<S>::value;
    return o;
  }
};

template <class S, class R> Ops pick_lim(int order, int lim) {
  if (order == 1 || lim == LIM_NONE) return Impl<S, R, 1, LIM_NONE>::ops();
  switch (lim) {
    case LIM_MINMOD: return Impl<S, R, 2, LIM_MINMOD>::ops();
    case LIM_SUPERBEE: return Impl<S, R, 2, LIM_SUPERBEE>::ops();
    default: return Impl<S, R, 2, LIM_MC>::ops();
  }
}

// per-solver factories, one translation unit each (ws_inst_*.cu), so the
// heavy template instantiations compile in parallel
Ops ops_acoustics_const(int prec, int order, int lim);
Ops ops_acoustics_var(int prec, int order, int lim);
Ops ops_euler_roe(int prec, int order, int lim);
Ops ops_euler_hlle(int prec, int order, int lim);
Ops ops_shallow_roe(int prec, int order, int lim);
Ops ops_f32_shallow_roe(int order, int lim);   // ws_inst_f32_shallow_roe.cu
Ops ops_advection(int prec, int order, int lim);
// WS_FP32_FAST: Fast<S> kernels from ws_inst_fast_*.cu (own compiler flags)
Ops ops_fast_acoustics_const(int order, int lim);
Ops ops_fast_acoustics_var(int order, int lim);
Ops ops_fast_euler_roe(int order, int lim);
Ops ops_fast_euler_hlle(int order, int lim);
Ops ops_fast_shallow_roe(int order, int lim);
Ops ops_fast_advection(int order, int lim);

// batched pointwise plugin call (ws_riemann), fp64
int riemann_acoustics_const(const double* p, int dir, long long n, const double* ql,
                            const double* qr, const double* al, const double* ar, double* w,
                            double* s, double* am, double* ap, int* codes);
int riemann_acoustics_var(const double* p, int dir, long long n, const double* ql,
                          const double* qr, const double* al, const double* ar, double* w,
                          double* s, double* am, double* ap, int* codes);
int riemann_euler_roe(const double* p, int dir, long long n, const double* ql, const double* qr,
                      const double* al, const double* ar, double* w, double* s, double* am,
                      double* ap, int* codes);
int riemann_euler_hlle(const double* p, int dir, long long n, const double* ql,
                       const double* qr, const double* al, const double* ar, double* w,
                       double* s, double* am, double* ap, int* codes);
int riemann_shallow_roe(const double* p, int dir, long long n, const double* ql,
                        const double* qr, const double* al, const double* ar, double* w,
                        double* s, double* am, double* ap, int* codes);
int riemann_advection(const double* p, int dir, long long n, const double* ql,
                      const double* qr, const double* al, const double* ar, double* w,
                      double* s, double* am, double* ap, int* codes);

template <class S>
int riemann_t(const typename S::template Params<double>& P, int dir, long long n,
              const double* ql, const double* qr, const double* al, const double* ar,
              double* waves, double* speeds, double* amdq, double* apdq, int* codes) {
  constexpr int NEQ = S::NEQ, NW = S::NW, NAUX = S::NAUX;
  if (NAUX > 0 && (!al || !ar)) return fail(nullptr, WS_ERR_CONFIG, "this solver needs aux data");
  const size_t b = sizeof(double) * (size_t)n;
  double *dql, *dqr, *dal = nullptr, *dar = nullptr, *dw, *ds, *dm, *dp;
  int* dc;
  cudaError_t e;
  std::vector<void*> bufs;
  auto alloc = [&](void** p, size_t bytes) {
    e = cudaMalloc(p, bytes > 0 ? bytes : 8);
    if (e == cudaSuccess) bufs.push_back(*p);
    return e == cudaSuccess;
  };
  auto cleanup = [&]() { for (void* p : bufs) cudaFree(p); };
  bool ok = alloc((void**)&dql, b * NEQ) && alloc((void**)&dqr, b * NEQ) &&
            alloc((void**)&dw, b * NW * NEQ) && alloc((void**)&ds, b * NW) &&
            alloc((void**)&dm, b * NEQ) && alloc((void**)&dp, b * NEQ) &&
            alloc((void**)&dc, sizeof(int) * (size_t)(n > 0 ? n : 1));
  if (ok && NAUX > 0) ok = alloc((void**)&dal, b * NAUX) && alloc((void**)&dar, b * NAUX);
  if (!ok) { cleanup(); return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e)); }
  cudaMemcpy(dql, ql, b * NEQ, cudaMemcpyHostToDevice);
  cudaMemcpy(dqr, qr, b * NEQ, cudaMemcpyHostToDevice);
  if (NAUX > 0) {
    cudaMemcpy(dal, al, b * NAUX, cudaMemcpyHostToDevice);
    cudaMemcpy(dar, ar, b * NAUX, cudaMemcpyHostToDevice);
  }
  if (n > 0) {
    const int blocks = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
    if (dir == 0)
      k_riemann<S, double, 1><<<blocks, 256>>>(P, n, dql, dqr, dal, dar, dw, ds, dm, dp, dc);
    else
      k_riemann<S, double, 2><<<blocks, 256>>>(P, n, dql, dqr, dal, dar, dw, ds, dm, dp, dc);
  }
  e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(waves, dw, b * NW * NEQ, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(speeds, ds, b * NW, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(amdq, dm, b * NEQ, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(apdq, dp, b * NEQ, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(codes, dc, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost);
  cleanup();
  if (e != cudaSuccess) return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e));
  return WS_OK;
}


}  // namespace wsh
