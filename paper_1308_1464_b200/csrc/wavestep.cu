// wavestep.cu — C-ABI implementation (include/wavestep.h).
//
// One handle = one shard of the grid on one GPU: ping-pong state buffers,
// aux, the device step state (reductions, reports, errors) and a stream.
// ws_step enqueues the CFL pre-pass (dynamic-speed solvers) and the fused
// update kernel without any host synchronisation; ws_run replays a captured
// two-step CUDA graph.  The translation unit is compiled with --fmad=false
// (bitwise parity with the numpy oracle, see ws_solvers.cuh).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ws_host.cuh"

using namespace wsh;

namespace {
thread_local std::string g_create_error;
}

int wsh::fail(ws_handle* h, int code, const std::string& msg) {
  if (h) h->err = msg; else g_create_error = msg;
  return code;
}

namespace {

template <class R> bool bind(ws_handle* h, std::string& msg) {
  const ws_desc& d = h->d;
  const double* p = d.params;
  switch (d.solver) {
    case WS_ACOUSTICS_CONST: {
      // reference kernels.py:106-118: both positive; c = sqrt(K/rho), Z = rho*c
      if (!(p[0] > 0 && p[1] > 0)) {
        char b[160];
        snprintf(b, sizeof b, "density and bulk modulus must be positive, got %.17g, %.17g",
                 p[0], p[1]);
        msg = b;
        return false;
      }
      double c = std::sqrt(p[1] / p[0]);
      double z = p[0] * c;
      AcousticsConst::Params<R> pr{(R)z, (R)(2.0 * z), (R)c};
      h->params.assign((char*)&pr, (char*)&pr + sizeof pr);
      h->host_static[0] = h->host_static[1] = (double)(R)c;
      h->ops = ops_acoustics_const(d.precision, d.order, d.limiter);
      h->neq = 3; h->naux = 0;
      return true;
    }
    case WS_ACOUSTICS_VAR: {
      AcousticsVar::Params<R> pr{(R)0};
      h->params.assign((char*)&pr, (char*)&pr + sizeof pr);
      h->ops = ops_acoustics_var(d.precision, d.order, d.limiter);
      h->neq = 3; h->naux = 2;
      return true;
    }
    case WS_EULER_ROE:
    case WS_EULER_HLLE: {
      if (!(p[0] > 1.0)) {
        char b[96];
        snprintf(b, sizeof b, "gamma must exceed 1, got %.17g", p[0]);
        msg = b;
        return false;
      }
      if (d.solver == WS_EULER_ROE) {
        EulerRoe::Params<R> pr{(R)(p[0] - 1.0)};
        h->params.assign((char*)&pr, (char*)&pr + sizeof pr);
        h->ops = ops_euler_roe(d.precision, d.order, d.limiter);
      } else {
        EulerHLLE::Params<R> pr{(R)(p[0] - 1.0), (R)p[0]};
        h->params.assign((char*)&pr, (char*)&pr + sizeof pr);
        h->ops = ops_euler_hlle(d.precision, d.order, d.limiter);
      }
      h->neq = 4; h->naux = 0;
      return true;
    }
    case WS_ADVECTION: {
      // reference kernels.py:169-170: non-finite velocity is a KernelError
      if (!(std::isfinite(p[0]) && std::isfinite(p[1]))) {
        char b[128];
        snprintf(b, sizeof b, "non-finite advection velocity (%.17g, %.17g)", p[0], p[1]);
        msg = b;
        return false;
      }
      Advection::Params<R> pr{(R)p[0], (R)p[1]};
      h->params.assign((char*)&pr, (char*)&pr + sizeof pr);
      h->host_static[0] = std::fabs((double)(R)p[0]);
      h->host_static[1] = std::fabs((double)(R)p[1]);
      h->ops = ops_advection(d.precision, d.order, d.limiter);
      h->neq = 1; h->naux = 0;
      return true;
    }
    case WS_SHALLOW_ROE: {
      if (!(p[0] > 0)) {
        char b[96];
        snprintf(b, sizeof b, "gravity must be positive, got %.17g", p[0]);
        msg = b;
        return false;
      }
      ShallowRoe::Params<R> pr{(R)p[0], (R)std::sqrt(p[0])};
      h->params.assign((char*)&pr, (char*)&pr + sizeof pr);
      h->ops = ops_shallow_roe(d.precision, d.order, d.limiter);
      h->neq = 3; h->naux = 0;
      return true;
    }
  }
  msg = "unknown solver id " + std::to_string(d.solver);
  return false;
}

long long pitch_for(int nx, size_t esz) {
  // 256-byte aligned component rows (coalescing; TMA-compatible strides)
  long long per = 256 / (long long)esz;
  return ((long long)nx + per - 1) / per * per;
}

int validate(const ws_desc* d, std::string& m) {
  char b[200];
  if (d->nx < 1 || d->ny < 1) {
    snprintf(b, sizeof b, "cell counts must be >= 1, got nx=%d, ny=%d", d->nx, d->ny);
    m = b; return WS_ERR_CONFIG;
  }
  if (!(d->dx > 0 && d->dy > 0)) {
    snprintf(b, sizeof b, "cell widths must be > 0, got dx=%.17g, dy=%.17g", d->dx, d->dy);
    m = b; return WS_ERR_CONFIG;
  }
  if (d->num_ghost != 2) {
    snprintf(b, sizeof b, "the device layout uses num_ghost=2, got %d", d->num_ghost);
    m = b; return WS_ERR_CONFIG;
  }
  if (d->order != 1 && d->order != 2) {
    snprintf(b, sizeof b, "order must be 1 or 2, got %d", d->order);
    m = b; return WS_ERR_CONFIG;
  }
  if (d->limiter < 0 || d->limiter > 3) { m = "unknown limiter"; return WS_ERR_CONFIG; }
  if ((d->bc_x != 0 && d->bc_x != 1) || (d->bc_y != 0 && d->bc_y != 1)) {
    m = "unknown boundary condition"; return WS_ERR_CONFIG;
  }
  if (d->precision != WS_FP64 && d->precision != WS_FP32 && d->precision != WS_FP32_FAST) {
    m = "unknown precision"; return WS_ERR_CONFIG;
  }
  // reference grid.py:165-169 (PERIODIC needs n >= num_ghost)
  if (d->bc_x == WS_BC_PERIODIC && d->nx < 2) {
    snprintf(b, sizeof b, "periodic boundary needs at least num_ghost=2 interior cells, got %d",
             d->nx);
    m = b; return WS_ERR_CONFIG;
  }
  bool multi = d->rows_lo == WS_ROWS_MEMORY || d->rows_hi == WS_ROWS_MEMORY;
  if (!multi && d->bc_y == WS_BC_PERIODIC && d->ny < 2) {
    snprintf(b, sizeof b, "periodic boundary needs at least num_ghost=2 interior cells, got %d",
             d->ny);
    m = b; return WS_ERR_CONFIG;
  }
  if (multi && d->ny < 2) { m = "a row-strip shard needs at least 2 rows"; return WS_ERR_CONFIG; }
  if (d->ny_global < d->ny || d->j_offset < 0 || d->j_offset + d->ny > d->ny_global) {
    m = "inconsistent row-strip geometry (ny_global / j_offset)"; return WS_ERR_CONFIG;
  }
  if (d->nx >= (1 << 19) || d->ny_global >= (1 << 18)) {
    m = "grid too large for the interface indices of the error key (nx < 2^19, ny < 2^18)";
    return WS_ERR_CONFIG;
  }
  return WS_OK;
}

void compute_layout(ws_handle* h) {
  const ws_desc& d = h->d;
  Layout& L = h->L;
  L.nx = d.nx; L.ny = d.ny;
  bool top = d.j_offset + d.ny == d.ny_global;
  L.ny_edges_y = d.ny + (top ? 1 : 0);
  L.bcx = d.bc_x; L.bcy = d.bc_y;
  L.lo = d.rows_lo == WS_ROWS_MEMORY ? ROWS_MEMORY : ROWS_BC;
  L.hi = d.rows_hi == WS_ROWS_MEMORY ? ROWS_MEMORY : ROWS_BC;
  L.j_off = d.j_offset;
  L.nx_glob = d.nx;
  L.trace = nullptr;
  L.trace_cap = 0;
  L.chk = nullptr;
  L.peers = nullptr;
  L.npeers = 0;
  L.nq_lo[0] = L.nq_lo[1] = L.nq_hi[0] = L.nq_hi[1] = nullptr;
  L.nds_lo = L.nds_hi = nullptr;
  L.ny_lo = 0;
  L.hsides = 0;
  L.pitch = pitch_for(d.nx, h->esz);
  L.rstride = (long long)h->neq * L.pitch;
  L.astride = (long long)h->naux * L.pitch;
}

StepArgs make_args(ws_handle* h, const ws_ctl* c, int cur) {
  StepArgs a{};
  a.dx = h->d.dx; a.dy = h->d.dy;
  a.cfl = c->cfl;
  a.has_dt_max = !std::isnan(c->dt_max); a.dt_max = c->dt_max;
  a.has_fixed = !std::isnan(c->fixed_dt); a.fixed_dt = c->fixed_dt;
  a.has_remaining = !std::isnan(c->remaining); a.remaining = c->remaining;
  a.has_t_final = !std::isnan(c->t_final); a.t_final = c->t_final;
  a.tol = a.has_t_final ? 1e-14 * std::fmax(1.0, c->t_final) : 0.0;   // driver.py:245
  a.cur = cur;
  a.static_speeds = (h->ops.static_speeds && !h->multi) ? 1 : 0;
  a.borders = h->borders;
  a.tmax = h->tile_prepass ? h->tmax : nullptr;
  return a;
}

int check_ctl(ws_handle* h, const ws_ctl* c) {
  // reference TimestepController.__post_init__, driver.py:25-31
  char b[128];
  if (!(c->cfl > 0.0 && c->cfl < 1.0)) {
    snprintf(b, sizeof b, "cfl_target must lie in (0, 1), got %.17g", c->cfl);
    return fail(h, WS_ERR_CONFIG, b);
  }
  if (!std::isnan(c->dt_max) && !(c->dt_max > 0)) return fail(h, WS_ERR_CONFIG, "dt_max must be positive");
  if (!std::isnan(c->fixed_dt) && !(c->fixed_dt > 0)) return fail(h, WS_ERR_CONFIG, "fixed_dt must be positive");
  return WS_OK;
}

// enqueue one step of parity `cur` from q[cur] into q[cur^1]
void enqueue_step(ws_handle* h, const ws_ctl* c, int cur, cudaStream_t st) {
  StepArgs a = make_args(h, c, cur);
  if (!a.static_speeds) {
    // fused mode: the pre-pass only for a state the epilogue has not probed
    if (!h->fused || h->need_prepass) h->ops.speeds(h, h->q[cur], cur, 0, st);
    h->need_prepass = false;
  }
  h->ops.update(h, h->q[cur], h->q[cur ^ 1], a, st);
}

}  // namespace

// ===========================================================================
extern "C" {

int ws_abi_version(void) { return WS_ABI_VERSION; }

int ws_buffer_bytes(const ws_desc* d, uint64_t* q_bytes, uint64_t* aux_bytes,
                    uint64_t* slots_bytes) {
  std::string m;
  int rc = validate(d, m);
  if (rc) return fail(nullptr, rc, m);
  size_t esz = d->precision == WS_FP64 ? 8 : 4;
  int neq = (d->solver == WS_EULER_ROE || d->solver == WS_EULER_HLLE) ? 4
            : (d->solver == WS_ADVECTION ? 1 : 3);
  int naux = d->solver == WS_ACOUSTICS_VAR ? 2 : 0;
  long long pitch = pitch_for(d->nx, esz);
  if (q_bytes) *q_bytes = (uint64_t)(d->ny + 4) * neq * pitch * esz;
  if (aux_bytes) *aux_bytes = (uint64_t)(d->ny + 4) * naux * pitch * esz;
  if (slots_bytes) *slots_bytes = sizeof(DevState);
  return WS_OK;
}

int ws_create(const ws_desc* d, ws_handle** out) {
  if (!d || !out) return fail(nullptr, WS_ERR_CONFIG, "null argument");
  *out = nullptr;
  std::string m;
  int rc = validate(d, m);
  if (rc) return fail(nullptr, rc, m);
  ws_handle* h = new ws_handle();
  h->d = *d;
  h->esz = d->precision == WS_FP64 ? 8 : 4;
  h->multi = d->rows_lo == WS_ROWS_MEMORY || d->rows_hi == WS_ROWS_MEMORY;
  bool ok = d->precision == WS_FP64 ? bind<double>(h, m) : bind<float>(h, m);
  if (!ok) { delete h; return fail(nullptr, WS_ERR_CONFIG, m); }
  compute_layout(h);
  cudaError_t e = cudaSetDevice(d->device);
  if (e != cudaSuccess) { delete h; return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e)); }
  uint64_t qb, ab, sb;
  ws_buffer_bytes(d, &qb, &ab, &sb);
  auto get = [&](void* ext, size_t bytes, void** dst, bool* own) -> cudaError_t {
    if (bytes == 0) { *dst = nullptr; *own = false; return cudaSuccess; }
    if (ext) { *dst = ext; *own = false; return cudaSuccess; }
    *own = true;
    return cudaMalloc(dst, bytes);
  };
  void* dsp = nullptr;
  if ((e = get(d->ext_q0, qb, &h->q[0], &h->own_q[0])) != cudaSuccess ||
      (e = get(d->ext_q1, qb, &h->q[1], &h->own_q[1])) != cudaSuccess ||
      (e = get(d->ext_aux, ab, &h->aux, &h->own_aux)) != cudaSuccess ||
      (e = get(d->ext_slots, sb, &dsp, &h->own_ds)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&h->ev_order, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&h->ev_in[0], cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&h->ev_in[1], cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&h->ev_copy[0], cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&h->ev_copy[1], cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming)) != cudaSuccess) {
    ws_destroy(h);
    return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e));
  }
  h->ds = static_cast<DevState*>(dsp);
  // fused next-step CFL epilogue: correct (bitwise) but slower than the
  // pre-pass on B200 in round 1 (profiles/r1_exp_fused.md) -> opt-in
  // fused next-step CFL epilogues (line kernel: in-tile probes + tile-border
  // kernel; tile kernel: shared-border counters) are bitwise correct but not
  // faster than the k_speeds pre-pass on B200 (profiles/r1_exp_fused.md):
  // opt-in with WS_FUSE=1
  h->line_kernel = true;          // warp-line kernel for every solver (WS_KERNEL=tile: tile kernel)
  if (const char* v = std::getenv("WS_KERNEL")) h->line_kernel = std::strcmp(v, "tile") != 0;
  if (const char* v = std::getenv("WS_SPEEDS")) {
    h->speeds_smem = std::strcmp(v, "smem") == 0;
    h->speeds_exact = std::strcmp(v, "exact") == 0;   // no candidate filter
    h->speeds_edge = std::strcmp(v, "edge") == 0;     // per-edge filter (k_speeds_b)
  }
  if (const char* v = std::getenv("WS_PDL")) h->pdl = std::atoi(v) != 0;
  if (const char* v = std::getenv("WS_PERSIST")) h->persist = std::atoi(v) != 0;
  if (const char* v = std::getenv("WS_RUN_SMALL")) h->run_small = std::atoi(v) != 0;
  {
    const char* v = std::getenv("WS_FUSE");
    const bool env_on = v && std::atoi(v) != 0, env_off = v && std::atoi(v) == 0;
    (void)env_off;
    if (h->line_kernel) h->fused = h->ops.can_fuse_line && !h->multi && env_on;
    else h->fused = !h->ops.static_speeds && !h->multi && env_on;
  }
  // generous for every tile shape (TX >= 16, TY >= 4): vertical + horizontal borders
  h->border_bytes = sizeof(int) * 2 * (size_t)((d->nx + 15) / 16 + 1) * ((d->ny + 3) / 4 + 1);
  if ((e = cudaMalloc(&h->borders, h->border_bytes)) != cudaSuccess) {
    ws_destroy(h);
    return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e));
  }
  cudaMemsetAsync(h->borders, 0, h->border_bytes, h->stream);
  // whole-tile CFL pre-pass (k_speeds_t): the update stores per-tile bound
  // maxima of the state it writes, the next pre-pass skips tiles that cannot
  // hold the step's maximum (WS_SPEEDS=exact|edge|smem select the others)
  // (a static-speed solver needs it only as a row-strip shard: its single
  // domain checks admissibility inside the update)
  h->tile_prepass = h->ops.tile_prepass && h->line_kernel && !h->fused &&
                    !h->speeds_exact && !h->speeds_smem && !h->speeds_edge &&
                    (!h->ops.static_speeds || h->multi);
  if (h->tile_prepass) {
    const size_t nt = (size_t)((d->nx + 28) / 29) * ((d->ny + 28) / 29);
    // [2][nt][nacc] int tile accumulators (S::tile_acc), one set per state buffer
    if ((e = cudaMalloc(&h->tmax, 2 * nt * 4 * (size_t)h->ops.nacc)) != cudaSuccess) {
      ws_destroy(h);
      return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e));
    }
  }
  h->ops.prepare();
  if (WS_CHECKED) {
    const size_t cb = sizeof(unsigned) * (1 + (size_t)d->nx * d->ny);
    if ((e = cudaMalloc(&h->chk, cb)) != cudaSuccess) {
      ws_destroy(h);
      return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e));
    }
    cudaMemsetAsync(h->chk, 0, cb, h->stream);
    h->L.chk = h->chk;
  }
  if (const char* v = std::getenv("WS_TRACE")) {
    if (std::atoi(v) != 0) {
      // diagnostics: one {start, end, smid, block} record per CTA of the pre-pass
      // (region 0) and the update kernel (region 1), overwritten every launch
      const long long cap = ((long long)(d->nx + 31) / 29 + 1) * ((d->ny + 31) / 16 + 1);
      if (cudaMalloc(&h->trace, sizeof(unsigned long long) * 8 * cap) == cudaSuccess) {
        cudaMemsetAsync(h->trace, 0, sizeof(unsigned long long) * 8 * cap, h->stream);
        h->L.trace = h->trace;
        h->L.trace_cap = (int)cap;
      }
    }
  }
  // zero everything once so ghost rows / padding are defined
  cudaMemsetAsync(h->q[0], 0, qb, h->stream);
  cudaMemsetAsync(h->q[1], 0, qb, h->stream);
  if (h->aux) cudaMemsetAsync(h->aux, 0, ab, h->stream);
  cudaMemsetAsync(h->ds, 0, sb, h->stream);
  e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) { ws_destroy(h); return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e)); }
  *out = h;
  return WS_OK;
}

void ws_destroy(ws_handle* h) {
  if (!h) return;
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  for (int k = 0; k < 2; ++k) if (h->own_q[k] && h->q[k]) cudaFree(h->q[k]);
  if (h->own_aux && h->aux) cudaFree(h->aux);
  if (h->own_ds && h->ds) cudaFree(h->ds);
  for (int k = 0; k < 2; ++k) if (h->stage[k]) cudaFree(h->stage[k]);
  if (h->stage_out) cudaFree(h->stage_out);
  if (h->stage_aux) cudaFree(h->stage_aux);
  if (h->peers_dev) cudaFree(h->peers_dev);
  if (h->ev_order) cudaEventDestroy(h->ev_order);
  for (int k = 0; k < 2; ++k) {
    if (h->ev_in[k]) cudaEventDestroy(h->ev_in[k]);
    if (h->ev_copy[k]) cudaEventDestroy(h->ev_copy[k]);
  }
  if (h->ev_out) cudaEventDestroy(h->ev_out);
  if (h->borders) cudaFree(h->borders);
  if (h->tmax) cudaFree(h->tmax);
  if (h->trace) cudaFree(h->trace);
  if (h->chk) cudaFree(h->chk);
  if (h->cstream) { cudaStreamSynchronize(h->cstream); cudaStreamDestroy(h->cstream); }
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

const char* ws_last_error(const ws_handle* h) {
  return h ? h->err.c_str() : g_create_error.c_str();
}

static int ensure_buf(ws_handle* h, void** buf, size_t* have, size_t bytes) {
  if (*have >= bytes) return WS_OK;
  if (*buf) { cudaDeviceSynchronize(); cudaFree(*buf); *buf = nullptr; }
  WS_CUDA(h, cudaMalloc(buf, bytes));
  *have = bytes;
  return WS_OK;
}

static int ensure_stage(ws_handle* h, int b, size_t bytes) {
  return ensure_buf(h, &h->stage[b], &h->stage_bytes[b], bytes);
}

static int upload_impl(ws_handle* h, const void* qh, const void* ah, size_t hesz, void* s) {
  if (!h || !qh) return fail(h, WS_ERR_CONFIG, "null argument");
  if (hesz != h->esz) return fail(h, WS_ERR_CONFIG, "host precision does not match the handle");
  if (h->naux > 0 && !ah) return fail(h, WS_ERR_CONFIG, "this solver needs aux data");
  const size_t cells = (size_t)(h->d.nx + 4) * (h->d.ny + 4);
  int ncmax = h->neq > h->naux ? h->neq : h->naux;
  // Two staging buffers, alternating, filled on the handle's copy stream: the
  // H2D of this upload waits only for the conversion of the upload before
  // the previous one, so it overlaps a step and a download still in flight
  // (PCIe is full duplex).  The conversion into the state runs on the
  // caller's stream after everything issued before (pick) and after the H2D.
  const int b = h->up_idx;
  h->up_idx ^= 1;
  int rc = ensure_stage(h, b, cells * ncmax * h->esz);
  if (rc) return rc;
  WS_CUDA(h, cudaStreamWaitEvent(h->cstream, h->ev_in[b], 0));
  WS_CUDA(h, cudaMemcpyAsync(h->stage[b], qh, cells * h->neq * h->esz, cudaMemcpyHostToDevice,
                             h->cstream));
  WS_CUDA(h, cudaEventRecord(h->ev_copy[b], h->cstream));
  cudaStream_t st = pick(h, s);
  WS_CUDA(h, cudaStreamWaitEvent(st, h->ev_copy[b], 0));
  h->ops.to_soa(h, h->stage[b], h->q[0], h->neq, st);
  if (h->naux > 0) {
    WS_CUDA(h, cudaMemcpyAsync(h->stage[b], ah, cells * h->naux * h->esz, cudaMemcpyHostToDevice, st));
    h->ops.to_soa(h, h->stage[b], h->aux, h->naux, st);
  }
  WS_CUDA(h, cudaEventRecord(h->ev_in[b], st));
  if (WS_CHECKED && h->chk) {
    WS_CUDA(h, cudaMemsetAsync(h->chk, 0, sizeof(unsigned) * (1 + (size_t)h->d.nx * h->d.ny), st));
    h->ops.canary(h, st);
  }
  WS_CUDA(h, cudaMemsetAsync(h->ds, 0, offsetof(DevState, rep), st));
  WS_CUDA(h, cudaMemsetAsync(h->borders, 0, h->border_bytes, st));
  h->need_prepass = true;
  if (h->ops.static_speeds) {
    if (h->naux > 0) {
      h->ops.static_speed(h, st);
    } else {
      unsigned long long b[2];
      for (int k = 0; k < 2; ++k) {
        if (h->esz == 8) { std::memcpy(&b[k], &h->host_static[k], 8); }
        else { float f = (float)h->host_static[k]; unsigned u; std::memcpy(&u, &f, 4); b[k] = u; }
      }
      // pageable source: synchronous w.r.t. the host, ordered on st
      WS_CUDA(h, cudaMemcpyAsync(&h->ds->static_bits[0], b, sizeof b, cudaMemcpyHostToDevice, st));
      WS_CUDA(h, cudaStreamSynchronize(st));
    }
  }
  WS_CUDA(h, launch_status(h));
  h->enq = 0;
  h->nrep_seen = 0;
  h->tf_pending = false;
  h->uploaded = true;
  return WS_OK;
}

int ws_upload(ws_handle* h, const double* q, const double* a, void* s) {
  return upload_impl(h, q, a, 8, s);
}
int ws_upload_f32(ws_handle* h, const float* q, const float* a, void* s) {
  return upload_impl(h, q, a, 4, s);
}

// host view of the DevState header
struct HostState {
  long long steps, err_step, nrep;
  unsigned long long err_key;
  int err, finished;
  double t;
};

static int read_state(ws_handle* h, HostState* hs, cudaStream_t st) {
  DevState tmp;
  WS_CUDA(h, cudaStreamSynchronize(st));
  if (h->stream != st) WS_CUDA(h, cudaStreamSynchronize(h->stream));
  WS_CUDA(h, cudaMemcpy(&tmp, h->ds, offsetof(DevState, rep), cudaMemcpyDeviceToHost));
  hs->steps = tmp.steps; hs->err_step = tmp.err_step; hs->nrep = tmp.nrep;
  hs->err_key = tmp.err_key; hs->err = tmp.err; hs->finished = tmp.finished; hs->t = tmp.t;
  return WS_OK;
}

// after a sync: re-align the enqueue counter with what the device committed
static int resync(ws_handle* h, const HostState& hs, cudaStream_t st) {
  if (h->enq != hs.steps) {
    h->enq = hs.steps;
    WS_CUDA(h, cudaMemsetAsync(&h->ds->slot[0][0], 0, sizeof(h->ds->slot), st));
    h->need_prepass = true;
  }
  return WS_OK;
}

static int download_impl(ws_handle* h, void* qh, size_t hesz, void* s, bool wait) {
  if (!h || !qh) return fail(h, WS_ERR_CONFIG, "null argument");
  if (hesz != h->esz) return fail(h, WS_ERR_CONFIG, "host precision does not match the handle");
  cudaStream_t st = pick(h, s);
  long long steps = h->enq;
  bool err = false;
  int rc;
  if (wait) {
    HostState hs;
    if ((rc = read_state(h, &hs, st))) return rc;
    if ((rc = resync(h, hs, st))) return rc;
    steps = hs.steps;
    err = hs.err != 0;
  }
  // (async: the host's count of enqueued steps stands in for the device's;
  // the caller checks ws_poll before trusting the array)
  const int cur = (int)(steps & 1);
  // ghosts hold the BC fill of the state the last (attempted) step started from
  const void* gsrc = (steps == 0 || err) ? h->q[cur] : h->q[cur ^ 1];
  const size_t bytes = (size_t)(h->d.nx + 4) * (h->d.ny + 4) * h->neq * h->esz;
  if ((rc = ensure_buf(h, &h->stage_out, &h->stage_out_bytes, bytes))) return rc;
  WS_CUDA(h, cudaStreamWaitEvent(st, h->ev_out, 0));   // previous copy-out done
  h->ops.to_aos(h, h->q[cur], gsrc, h->stage_out, st);
  // later operations on other streams order after the conversion, not after
  // the copy to the host (only the next download reuses stage_out, and it is
  // stream-ordered behind this copy when issued on the same stream)
  WS_CUDA(h, cudaEventRecord(h->ev_order, st));
  WS_CUDA(h, cudaMemcpyAsync(qh, h->stage_out, bytes, cudaMemcpyDeviceToHost, st));
  WS_CUDA(h, cudaEventRecord(h->ev_out, st));
  h->order_recorded = true;
  if (wait) WS_CUDA(h, cudaStreamSynchronize(st));
  return WS_OK;
}

int ws_download(ws_handle* h, double* q, void* s) { return download_impl(h, q, 8, s, true); }
int ws_download_f32(ws_handle* h, float* q, void* s) { return download_impl(h, q, 4, s, true); }
int ws_download_async(ws_handle* h, void* q, void* s) {
  return download_impl(h, q, h ? h->esz : 8, s, false);
}

// Steps pick their buffers from the host's count of enqueued steps.  A step
// whose control carries t_final can stop on the device (t reached), so after
// one the host count may run ahead of the committed steps.  Continuing with
// the same t_final is harmless (every further step is a no-op), anything else
// first re-aligns the count with the device and clears the finished flag.
static int tfinal_guard(ws_handle* h, const ws_ctl* c, cudaStream_t st) {
  const bool tf = !std::isnan(c->t_final);
  if (h->tf_pending && tf && c->t_final == h->tf_value) return WS_OK;
  if (h->tf_pending) {
    HostState hs;
    int rc = read_state(h, &hs, st);
    if (rc) return rc;
    if ((rc = resync(h, hs, st))) return rc;
    // only a t_final step sets the flag, and upload clears it
    WS_CUDA(h, cudaMemsetAsync(&h->ds->finished, 0, sizeof(int), st));
  }
  h->tf_pending = tf;
  h->tf_value = tf ? c->t_final : 0.0;
  return WS_OK;
}

int ws_download_aux_ghosts(ws_handle* h, void* ah, void* s) {
  if (!h || !ah) return fail(h, WS_ERR_CONFIG, "null argument");
  if (h->naux == 0) return WS_OK;
  if (!h->uploaded) return fail(h, WS_ERR_CONFIG, "no state uploaded");
  cudaStream_t st = pick(h, s);
  const long long nxt = h->d.nx + 4, nyt = h->d.ny + 4;
  const size_t es = h->esz, na = (size_t)h->naux;
  int rc = ensure_buf(h, &h->stage_aux, &h->stage_aux_bytes, (size_t)(nxt * nyt) * na * es);
  if (rc) return rc;
  h->ops.to_aos_aux(h, h->stage_aux, st);
  char* hd = static_cast<char*>(ah);
  const char* sd = static_cast<const char*>(h->stage_aux);
  const size_t row = (size_t)nxt * na * es;           // one j of the host layout
  // rows j = 0, 1 and j = ny+2, ny+3: contiguous
  WS_CUDA(h, cudaMemcpyAsync(hd, sd, 2 * row, cudaMemcpyDeviceToHost, st));
  const size_t top = (size_t)(nyt - 2) * row;
  WS_CUDA(h, cudaMemcpyAsync(hd + top, sd + top, 2 * row, cudaMemcpyDeviceToHost, st));
  // columns i = 0, 1 and i = nx+2, nx+3 of the interior rows: strided
  const size_t lo = 2 * row, hi = 2 * row + (size_t)(nxt - 2) * na * es;
  WS_CUDA(h, cudaMemcpy2DAsync(hd + lo, row, sd + lo, row, 2 * na * es, (size_t)h->d.ny,
                               cudaMemcpyDeviceToHost, st));
  WS_CUDA(h, cudaMemcpy2DAsync(hd + hi, row, sd + hi, row, 2 * na * es, (size_t)h->d.ny,
                               cudaMemcpyDeviceToHost, st));
  WS_CUDA(h, cudaStreamSynchronize(st));
  return WS_OK;
}

int ws_checked_counts(ws_handle* h, uint32_t* flags, uint32_t* wmin, uint32_t* wmax) {
  if (!h || !flags || !wmin || !wmax) return fail(h, WS_ERR_CONFIG, "null argument");
  if (!WS_CHECKED || !h->chk) return fail(h, WS_ERR_CONFIG, "not a checked build (-DWS_CHECKED=1)");
  cudaStream_t st = h->last_stream ? h->last_stream : h->stream;
  WS_CUDA(h, cudaStreamSynchronize(st));
  std::vector<unsigned> c(1 + (size_t)h->d.nx * h->d.ny);
  WS_CUDA(h, cudaMemcpy(c.data(), h->chk, sizeof(unsigned) * c.size(), cudaMemcpyDeviceToHost));
  unsigned lo = ~0u, hi = 0u;
  for (size_t k = 1; k < c.size(); ++k) { lo = c[k] < lo ? c[k] : lo; hi = c[k] > hi ? c[k] : hi; }
  *flags = c[0]; *wmin = lo; *wmax = hi;
  return WS_OK;
}

int ws_pin_host(void* p, uint64_t bytes) {
  if (!p || bytes == 0) return fail(nullptr, WS_ERR_CONFIG, "null or empty host range");
  cudaError_t e = cudaHostRegister(p, (size_t)bytes, cudaHostRegisterPortable);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e)); }
  return WS_OK;
}

int ws_unpin_host(void* p) {
  if (!p) return fail(nullptr, WS_ERR_CONFIG, "null host pointer");
  cudaError_t e = cudaHostUnregister(p);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e)); }
  return WS_OK;
}

// a row-strip shard can run whole steps only when the kernels do its
// collectives (slot reduction and every memory ghost-row side pushed)
static bool device_collectives(const ws_handle* h) {
  const int mem_sides = (h->L.lo == ROWS_MEMORY ? 1 : 0) + (h->L.hi == ROWS_MEMORY ? 1 : 0);
  return h->L.npeers > 0 && h->L.hsides == mem_sides;
}

static const char* kShardStepMsg =
    "a row-strip shard steps through ws_phase_speeds / ws_phase_update with the host "
    "exchanging halos and reducing the slot, or with ws_set_peers + ws_set_halo_peers";

int ws_step(ws_handle* h, const ws_ctl* c, void* s) {
  if (!h || !c) return fail(h, WS_ERR_CONFIG, "null argument");
  if (!h->uploaded) return fail(h, WS_ERR_CONFIG, "no state uploaded");
  if (h->multi && !device_collectives(h)) return fail(h, WS_ERR_CONFIG, kShardStepMsg);
  int rc = check_ctl(h, c);
  if (rc) return rc;
  cudaStream_t st = pick(h, s);
  if ((rc = tfinal_guard(h, c, st))) return rc;
  // a small static-speed grid: the step as one launch of k_run_small (one
  // 30-warp CTA per tile: a line per warp instead of three)
  const StepArgs a = make_args(h, c, (int)(h->enq & 1));
  if (!(a.static_speeds && h->ops.run_small(h, a, 1, st)))
    enqueue_step(h, c, (int)(h->enq & 1), st);
  h->enq++;
  WS_CUDA(h, launch_status(h));
  return WS_OK;
}

int ws_phase_speeds(ws_handle* h, void* s) { return ws_phase_speeds_part(h, 0, s); }

int ws_phase_speeds_part(ws_handle* h, int32_t part, void* s) {
  if (!h) return fail(h, WS_ERR_CONFIG, "null argument");
  if (part < 0 || part > 2) return fail(h, WS_ERR_CONFIG, "part must be 0, 1 or 2");
  cudaStream_t st = pick(h, s);
  if (part != 0 && (h->fused || (h->ops.static_speeds && !h->multi))) {
    // split pre-pass only exists for the dynamic-speed, unfused path (shards)
    return fail(h, WS_ERR_CONFIG, "split CFL pre-pass needs a dynamic-speed, unfused handle");
  }
  // single-shard dynamic solvers probe the next state in the update epilogue;
  // a static-speed single domain needs no pre-pass (speeds fixed at upload,
  // admissibility checked by the update: the whole-step path)
  if ((!h->fused || h->need_prepass) && !(h->ops.static_speeds && !h->multi))
    h->ops.speeds(h, h->q[h->enq & 1], (int)(h->enq & 1), part, st);
  if (part != 1) h->need_prepass = false;
  WS_CUDA(h, launch_status(h));
  return WS_OK;
}

int ws_phase_update(ws_handle* h, const ws_ctl* c, void* s) {
  if (!h || !c) return fail(h, WS_ERR_CONFIG, "null argument");
  int rc = check_ctl(h, c);
  if (rc) return rc;
  cudaStream_t st = pick(h, s);
  const int cur = (int)(h->enq & 1);
  StepArgs a = make_args(h, c, cur);
  h->ops.update(h, h->q[cur], h->q[cur ^ 1], a, st);
  h->enq++;
  WS_CUDA(h, launch_status(h));
  return WS_OK;
}

int ws_phase_update_part(ws_handle* h, const ws_ctl* c, int32_t part, void* s) {
  if (!h || !c) return fail(h, WS_ERR_CONFIG, "null argument");
  if (part == 0) return ws_phase_update(h, c, s);
  if (part != 1 && part != 2) return fail(h, WS_ERR_CONFIG, "part must be 0, 1 or 2");
  if (!h->line_kernel || h->fused)
    return fail(h, WS_ERR_CONFIG, "a split update needs the warp-line kernel without the fused epilogue");
  int rc = check_ctl(h, c);
  if (rc) return rc;
  cudaStream_t st = pick(h, s);
  const int cur = (int)(h->enq & 1);
  StepArgs a = make_args(h, c, cur);
  // the tile rows holding local rows {0, 1} and {ny-2, ny-1}: what the
  // neighbours read as ghost rows next step
  const int nty = (h->d.ny + 28) / 29;
  a.tr_lo = nty < 1 ? nty : 1;
  a.tr_hi = (h->d.ny - 2) / 29;
  if (a.tr_hi < a.tr_lo) a.tr_hi = a.tr_lo;
  a.part = 1;
  const int n1 = h->ops.update_ctas(h, a);
  a.part = 2;
  const int n2 = h->ops.update_ctas(h, a);
  a.nblk_total = n1 + n2;
  a.part = part;
  h->ops.update(h, h->q[cur], h->q[cur ^ 1], a, st);
  if (part == 2) h->enq++;
  WS_CUDA(h, launch_status(h));
  return WS_OK;
}

int ws_capture_begin(ws_handle* h) {
  if (!h) return fail(h, WS_ERR_CONFIG, "null argument");
  if (!h->uploaded) return fail(h, WS_ERR_CONFIG, "no state uploaded");
  if (h->cap_open) return fail(h, WS_ERR_CONFIG, "a capture is already open");
  h->cap_open = true;
  h->cap_enq = h->enq;
  h->cap_launches = h->launches;
  return WS_OK;
}

int ws_capture_end(ws_handle* h, int64_t* steps, int64_t* launches) {
  if (!h) return fail(h, WS_ERR_CONFIG, "null argument");
  if (!h->cap_open) return fail(h, WS_ERR_CONFIG, "no capture open");
  h->cap_open = false;
  const long long ds = h->enq - h->cap_enq, dl = h->launches - h->cap_launches;
  h->enq = h->cap_enq;
  h->launches = h->cap_launches;
  if (ds % 2 != 0)
    return fail(h, WS_ERR_CONFIG, "a captured graph must hold an even number of steps");
  if (steps) *steps = ds;
  if (launches) *launches = dl;
  return WS_OK;
}

int ws_replayed(ws_handle* h, int64_t steps, int64_t launches) {
  if (!h) return fail(h, WS_ERR_CONFIG, "null argument");
  if (steps < 0 || steps % 2 != 0 || launches < 0)
    return fail(h, WS_ERR_CONFIG, "replayed steps must be even and >= 0");
  h->enq += steps;
  h->launches += launches;
  return WS_OK;
}

void* ws_slot_ptr(ws_handle* h) { return h ? (void*)&h->ds->slot[h->enq & 1][0] : nullptr; }

int ws_halo_ptrs(ws_handle* h, void** slo, void** shi, void** rlo, void** rhi, uint64_t* bytes) {
  if (!h) return fail(h, WS_ERR_CONFIG, "null argument");
  char* b = static_cast<char*>(h->q[h->enq & 1]);
  const long long rs = h->L.rstride * (long long)h->esz;
  if (slo) *slo = b + 2 * rs;
  if (shi) *shi = b + (long long)h->L.ny * rs;
  if (rlo) *rlo = b;
  if (rhi) *rhi = b + (long long)(h->L.ny + 2) * rs;
  if (bytes) *bytes = (uint64_t)(2 * rs);
  return WS_OK;
}

int ws_state_ptr(ws_handle* h, void** q, int64_t* pitch, int64_t* row) {
  if (!h) return fail(h, WS_ERR_CONFIG, "null argument");
  if (q) *q = h->q[h->enq & 1];
  if (pitch) *pitch = h->L.pitch;
  if (row) *row = h->L.rstride;
  return WS_OK;
}

int ws_run(ws_handle* h, int32_t nsteps, const ws_ctl* c, void* s) {
  if (!h || !c) return fail(h, WS_ERR_CONFIG, "null argument");
  if (!h->uploaded) return fail(h, WS_ERR_CONFIG, "no state uploaded");
  if (nsteps < 0) return fail(h, WS_ERR_CONFIG, "nsteps must be >= 0");
  if (h->multi && !device_collectives(h)) return fail(h, WS_ERR_CONFIG, kShardStepMsg);
  int rc = check_ctl(h, c);
  if (rc) return rc;
  cudaStream_t st = pick(h, s);
  if ((rc = tfinal_guard(h, c, st))) return rc;
  long long left = nsteps;
  if (left >= 1) {
    // small static-speed grid: every step in one cooperative launch
    const StepArgs a = make_args(h, c, (int)(h->enq & 1));
    if (a.static_speeds && h->ops.run_small(h, a, (int)left, st)) { h->enq += left; left = 0; }
  }
  if (left > 0 && (h->enq & 1)) { enqueue_step(h, c, 1, st); h->enq++; left--; }
  if (left >= 4 && h->need_prepass && !h->ops.static_speeds) {
    // keep the one-off pre-pass out of the captured graph
    enqueue_step(h, c, 0, st); h->enq++; left--;
    enqueue_step(h, c, 1, st); h->enq++; left--;
  }
  // (shards with device collectives replay the same graph: the pushes their
  // kernels await are counted from DevState::seq on the device)
  if (left >= 4 && st != nullptr) {
    // two-step graph (parity 0 then 1), cached per (ctl, stream)
    if (!h->gexec || std::memcmp(&h->gctl, c, sizeof(ws_ctl)) != 0 || h->gstream != st) {
      if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; }
      cudaGraph_t g;
      long long l0 = h->launches;
      WS_CUDA(h, cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      enqueue_step(h, c, 0, st);
      enqueue_step(h, c, 1, st);
      WS_CUDA(h, cudaStreamEndCapture(st, &g));
      h->graph_launches = h->launches - l0;
      h->launches = l0;
      WS_CUDA(h, cudaGraphInstantiate(&h->gexec, g, 0));
      cudaGraphDestroy(g);
      h->gctl = *c;
      h->gstream = st;
    }
    while (left >= 2) {
      WS_CUDA(h, cudaGraphLaunch(h->gexec, st));
      h->launches += h->graph_launches;
      h->enq += 2;
      left -= 2;
    }
  }
  while (left > 0) { enqueue_step(h, c, (int)(h->enq & 1), st); h->enq++; left--; }
  WS_CUDA(h, launch_status(h));
  return WS_OK;
}

int ws_poll(ws_handle* h, int64_t* steps_done, ws_report* reports, int32_t max_reports,
            int32_t* n_reports, double* t_now, ws_error_info* err) {
  if (!h) return fail(h, WS_ERR_CONFIG, "null argument");
  cudaStream_t st = h->last_stream ? h->last_stream : h->stream;
  HostState hs;
  int rc = read_state(h, &hs, st);
  if (rc) return rc;
  if ((rc = resync(h, hs, st))) return rc;
  WS_CUDA(h, cudaStreamSynchronize(st));
  if (steps_done) *steps_done = hs.steps;
  if (t_now) *t_now = hs.t;
  long long avail = hs.nrep - h->nrep_seen;
  if (avail > REPCAP) avail = REPCAP;
  long long want = avail < max_reports ? avail : max_reports;
  if (n_reports) *n_reports = (int32_t)want;
  if (reports && want > 0) {
    std::vector<Report> tmp((size_t)want);
    long long first = hs.nrep - want;
    long long k = 0;
    while (k < want) {
      long long idx = (first + k) % REPCAP;
      long long n = want - k;
      if (idx + n > REPCAP) n = REPCAP - idx;
      WS_CUDA(h, cudaMemcpy(&tmp[(size_t)k], &h->ds->rep[idx], sizeof(Report) * n,
                            cudaMemcpyDeviceToHost));
      k += n;
    }
    for (long long m = 0; m < want; ++m) {
      reports[m].dt = tmp[m].dt; reports[m].cfl = tmp[m].cfl;
      reports[m].max_speed_x = tmp[m].msx; reports[m].max_speed_y = tmp[m].msy;
    }
  }
  h->nrep_seen = hs.nrep;
  if (err) {
    std::memset(err, 0, sizeof *err);
    err->code = hs.err;
    err->step = hs.err_step;
    if (hs.err == ERR_KERNEL) {
      unsigned long long k = hs.err_key;
      err->direction = (int)(k >> 62);
      err->stage = (int)((k >> 40) & 0xf);
      err->component = (int)((k >> 37) & 0x7);
      err->i = (int)((k >> 18) & 0x7ffff);
      err->j = (int)(k & 0x3ffff);
    }
  }
  return hs.err ? hs.err : WS_OK;
}

int ws_sync(ws_handle* h) {
  if (!h) return fail(h, WS_ERR_CONFIG, "null argument");
  cudaStream_t st = h->last_stream ? h->last_stream : h->stream;
  WS_CUDA(h, cudaStreamSynchronize(st));
  return WS_OK;
}

int64_t ws_launch_count(const ws_handle* h) { return h ? h->launches : 0; }

void* ws_devstate_ptr(ws_handle* h) { return h ? (void*)h->ds : nullptr; }

int ws_set_halo_peers(ws_handle* h, void* const* lo_q, void* lo_state, int32_t ny_lo,
                      void* const* hi_q, void* hi_state) {
  if (!h) return fail(h, WS_ERR_CONFIG, "null argument");
  const bool lo = lo_state != nullptr, hi = hi_state != nullptr;
  if ((lo && (!lo_q || !lo_q[0] || !lo_q[1] || ny_lo < 2)) || (hi && (!hi_q || !hi_q[0] || !hi_q[1])))
    return fail(h, WS_ERR_CONFIG, "halo peer: both state buffers, its DevState and ny >= 2");
  if ((lo && h->L.lo != ROWS_MEMORY) || (hi && h->L.hi != ROWS_MEMORY))
    return fail(h, WS_ERR_CONFIG, "halo peers only on sides whose ghost rows are in memory");
  if ((lo || hi) && (!h->line_kernel || h->fused))
    return fail(h, WS_ERR_CONFIG, "device-side halos need the warp-line update");
  h->L.nq_lo[0] = lo ? lo_q[0] : nullptr; h->L.nq_lo[1] = lo ? lo_q[1] : nullptr;
  h->L.nq_hi[0] = hi ? hi_q[0] : nullptr; h->L.nq_hi[1] = hi ? hi_q[1] : nullptr;
  h->L.nds_lo = static_cast<DevState*>(lo_state);
  h->L.nds_hi = static_cast<DevState*>(hi_state);
  h->L.ny_lo = lo ? ny_lo : 0;
  // pushes this shard receives per step: one per neighbour side it has
  h->L.hsides = (h->L.lo == ROWS_MEMORY && lo ? 1 : 0) + (h->L.hi == ROWS_MEMORY && hi ? 1 : 0);
  return WS_OK;
}

int ws_set_peers(ws_handle* h, int32_t npeers, void* const* peer_states) {
  if (!h) return fail(h, WS_ERR_CONFIG, "null argument");
  if (npeers < 0 || npeers > WS_MAX_PEERS || (npeers > 0 && !peer_states))
    return fail(h, WS_ERR_CONFIG, "npeers must lie in [0, 8] with a pointer table");
  if (npeers > 0 && (!h->line_kernel || h->fused || (h->ops.static_speeds && !h->multi)))
    return fail(h, WS_ERR_CONFIG,
                "device-side reduction needs the warp-line update with a CFL pre-pass");
  if (!h->peers_dev) WS_CUDA(h, cudaMalloc(&h->peers_dev, sizeof(void*) * WS_MAX_PEERS));
  if (npeers > 0) {
    WS_CUDA(h, cudaMemcpy(h->peers_dev, peer_states, sizeof(void*) * npeers,
                          cudaMemcpyHostToDevice));
  }
  h->L.peers = reinterpret_cast<DevState* const*>(h->peers_dev);
  h->L.npeers = npeers;
  return WS_OK;
}

int ws_trace(ws_handle* h, uint64_t* out, int64_t cap, int64_t* n) {
  if (!h || !out || !n) return WS_ERR_CONFIG;
  *n = 0;
  if (!h->trace) return WS_OK;
  const int64_t words = 8ll * h->L.trace_cap;
  const int64_t m = cap < words ? cap : words;
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e == cudaSuccess) e = cudaMemcpy(out, h->trace, sizeof(uint64_t) * m, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(h, e, "ws_trace");
  *n = m;
  return WS_OK;
}

}  // extern "C"

extern "C" {

int ws_riemann(int32_t solver, const double* p, int32_t direction, int64_t n, const double* ql,
               const double* qr, const double* al, const double* ar, double* waves,
               double* speeds, double* amdq, double* apdq, int32_t* codes, int32_t device) {
  if (n < 0 || !ql || !qr || !waves || !speeds || !amdq || !apdq || !codes || !p)
    return fail(nullptr, WS_ERR_CONFIG, "bad argument");
  if (direction != 0 && direction != 1) return fail(nullptr, WS_ERR_CONFIG, "direction must be 0 or 1");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e));
  switch (solver) {
    case WS_ACOUSTICS_CONST: {
      if (!(p[0] > 0 && p[1] > 0))
        return fail(nullptr, WS_ERR_CONFIG, "density and bulk modulus must be positive");
      double c = std::sqrt(p[1] / p[0]), z = p[0] * c;
      (void)z;
      return riemann_acoustics_const(p, direction, n, ql, qr, al, ar, waves, speeds, amdq,
                                     apdq, codes);
    }
    case WS_ACOUSTICS_VAR: {
      return riemann_acoustics_var(p, direction, n, ql, qr, al, ar, waves, speeds, amdq,
                                   apdq, codes);
    }
    case WS_EULER_ROE: {
      if (!(p[0] > 1.0)) return fail(nullptr, WS_ERR_CONFIG, "gamma must exceed 1");
      return riemann_euler_roe(p, direction, n, ql, qr, al, ar, waves, speeds, amdq, apdq,
                               codes);
    }
    case WS_EULER_HLLE: {
      if (!(p[0] > 1.0)) return fail(nullptr, WS_ERR_CONFIG, "gamma must exceed 1");
      return riemann_euler_hlle(p, direction, n, ql, qr, al, ar, waves, speeds, amdq, apdq,
                                codes);
    }
    case WS_ADVECTION:
      return riemann_advection(p, direction, n, ql, qr, al, ar, waves, speeds, amdq, apdq,
                               codes);
    case WS_SHALLOW_ROE: {
      if (!(p[0] > 0)) return fail(nullptr, WS_ERR_CONFIG, "gravity must be positive");
      return riemann_shallow_roe(p, direction, n, ql, qr, al, ar, waves, speeds, amdq, apdq,
                                 codes);
    }
  }
  return fail(nullptr, WS_ERR_CONFIG, "unknown solver id");
}

int ws_fill_ghost(double* data, int32_t ncomp, int32_t nx, int32_t ny, int32_t bcx, int32_t bcy,
                  int32_t device) {
  if (!data || ncomp < 0 || nx < 1 || ny < 1) return fail(nullptr, WS_ERR_CONFIG, "bad argument");
  if (ncomp == 0) return WS_OK;
  char b[128];
  if (bcx == WS_BC_PERIODIC && nx < 2) {
    snprintf(b, sizeof b, "periodic boundary needs at least num_ghost=2 interior cells, got %d", nx);
    return fail(nullptr, WS_ERR_CONFIG, b);
  }
  if (bcy == WS_BC_PERIODIC && ny < 2) {
    snprintf(b, sizeof b, "periodic boundary needs at least num_ghost=2 interior cells, got %d", ny);
    return fail(nullptr, WS_ERR_CONFIG, b);
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e));
  const size_t bytes = sizeof(double) * (size_t)ncomp * (nx + 4) * (ny + 4);
  double* d = nullptr;
  if ((e = cudaMalloc(&d, bytes)) != cudaSuccess) return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e));
  e = cudaMemcpy(d, data, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    k_fill_ghost<><<<148 * 4, 256>>>(d, ncomp, nx, ny, bcx, bcy);
    e = cudaMemcpy(data, d, bytes, cudaMemcpyDeviceToHost);
  }
  cudaFree(d);
  if (e != cudaSuccess) return fail(nullptr, WS_ERR_CUDA, cudaGetErrorString(e));
  return WS_OK;
}

}  // extern "C"
