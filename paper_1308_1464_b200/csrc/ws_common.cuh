// ws_common.cuh — device layout, boundary index mapping and step control
// shared by every kernel of the B200 wave-propagation step.
//
// Device storage: one buffer per state, rows j in [-2, ny+2)
// of the shard, each row holding the num_eqn component rows of `pitch`
// elements (x fastest).  Address of (component c, cell i, row j):
//     base + (j + 2) * rstride + c * pitch + i,   rstride = num_eqn * pitch.
// Only the interior columns are stored; x ghost cells and physical-boundary
// y ghost rows are produced by index mapping on load, which is exactly the
// reference fill_ghost (grid.py:156-193: extrapolate copies the nearest
// interior cell, periodic wraps).  The two ghost rows per side exist in
// memory for the row-strip halo exchange.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef WS_CHECKED
#define WS_CHECKED 0
#endif

namespace ws {

// Checked builds (-DWS_CHECKED=1, _lib/checked/): the device analogue of the
// reference's WAVESWEEP_CHECKED mode (sweep.py:32-33, 78-96, which counts
// writes per interface slot and asserts exactly one).  Every kernel checks
// its shared-memory and global indices against the layout, a broken check
// sets a bit in Layout::chk[0], and the update kernel counts its writes per
// interior cell in chk[1 + j*nx + i] (exactly one per step).  The upload
// also fills every location no kernel may read (padding columns, the ghost
// rows of physical boundaries) with NaN, so a stray read poisons the result
// that the parity tests compare bit for bit.
enum : unsigned {
  CHK_STAGE_SMEM = 1u, CHK_STAGE_READ = 2u, CHK_EDGE_SMEM = 4u, CHK_X_SMEM = 8u,
  CHK_STORE = 16u, CHK_PREPASS_READ = 32u, CHK_TILE_LIST = 64u
};
#define WS_CHK(L, cond, bit)                                                    \
  do {                                                                          \
    if (WS_CHECKED) {                                                           \
      if (!(cond) && (L).chk != nullptr) atomicOr((L).chk, (unsigned)(bit));   \
    }                                                                           \
  } while (0)

enum : int { BC_PERIODIC = 0, BC_EXTRAPOLATE = 1 };
enum : int { ROWS_MEMORY = 0, ROWS_BC = 1 };
enum : int { LIM_NONE = 0, LIM_MINMOD = 1, LIM_SUPERBEE = 2, LIM_MC = 3 };

constexpr int REPCAP = 4096;          // device report ring (steps between polls)
constexpr int ERR_KERNEL = 1;
constexpr int ERR_STATIONARY = 4;
constexpr int ERR_WAIT_TIMEOUT = 3;   // a device-side wait gave up (reported as WS_ERR_CUDA)
constexpr int ERR_INTERNAL = 5;       // a device-side invariant broke (reported as WS_ERR_CUDA)

struct DevState;

struct Layout {
  int nx, ny;             // local interior
  int ny_edges_y;         // y-edge rows this shard reports (ny, +1 on the top shard)
  int bcx, bcy;           // BC_*
  int lo, hi;             // ROWS_* for the bottom / top ghost rows
  int j_off;              // global index of local row 0
  int nx_glob;            // == nx (x is never split)
  long long pitch;        // elements per component row
  long long rstride;      // elements per grid row of q   (num_eqn * pitch)
  long long astride;      // elements per grid row of aux (num_aux * pitch)
  unsigned long long* trace;  // CTA timeline (WS_TRACE=1 diagnostics) or null
  int trace_cap;              // CTAs per traced kernel
  struct DevState* const* peers;  // device-side slot reduce: every shard's state (or null)
  int npeers;
  // device-side halo push: the neighbours' two state buffers (this GPU's
  // mapping), their DevState, the low neighbour's row count; null = none
  void* nq_lo[2];
  void* nq_hi[2];
  struct DevState* nds_lo;
  struct DevState* nds_hi;
  int ny_lo;
  int hsides;                 // ghost-row sides this shard receives by push (0..2)
  unsigned* chk;              // checked builds: {violation bits, write count per cell}
};

// a row a kernel may read after index mapping: memory ghost rows only on
// sides whose ghost rows are in memory, else interior rows
__device__ __forceinline__ bool row_readable(int j, const Layout& L) {
  return j >= (L.lo == ROWS_MEMORY ? -2 : 0) && j < L.ny + (L.hi == ROWS_MEMORY ? 2 : 0);
}

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may start before its predecessor in
// the stream finishes; griddepcontrol.wait blocks until the predecessor has
// completed and flushed, launch_dependents lets the successor launch once
// every CTA of this grid has issued it.  No-ops for plain launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// system-scope acquire load (peer GPUs write the counter over NVLink)
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// CTA timeline record (diagnostics): {start ns, end ns, smid, linear block}
// written by thread 0; region 0 = CFL pre-pass, region 1 = update kernel
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_cta(const Layout& L, int region, unsigned long long t0) {
  const int b = blockIdx.y * gridDim.x + blockIdx.x;
  if (L.trace == nullptr || b >= L.trace_cap) return;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  unsigned long long* r = L.trace + 4ull * ((unsigned long long)region * L.trace_cap + b);
  r[0] = t0; r[1] = gtimer(); r[2] = smid; r[3] = b;
}

struct Report { double dt, cfl, msx, msy; };

// Device-resident step state.  slot[k&1] = {max|s| x bits, max|s| y bits,
// NKEY_MAX - first error key}: every entry is reduced with MAX (non-negative
// IEEE values order like their bit patterns; the smallest key wins), which is
// also what a multi-shard all-reduce (int64 MAX) of the 3 words does.
struct DevState {
  unsigned long long slot[2][3];
  unsigned long long static_bits[2];  // acoustics: precomputed max speeds
  int err;                            // sticky status (ERR_*), 0 = fine
  int done;                           // last-block counter of the update kernel
  long long steps;                    // committed steps since upload
  long long err_step;
  unsigned long long err_key;
  double t;                           // simulated time since upload
  int finished;                       // t_final reached
  int pdone;                          // pre-pass CTA counter (device-side slot push)
  long long nrep;                     // reports written (ring index)
  unsigned long long arrive;          // slot pushes received from the shards (device reduce)
  unsigned long long harrive;         // halo-row pushes received from the neighbours
  unsigned long long mctr[2];         // k_run_small grid barrier per step parity:
                                      // arrivals (low 32) | arrivals with an error (high 32)
  long long seq;                      // update kernels committed since upload (skipped
                                      // steps too): the pushes a shard awaits are
                                      // counted from it on the device, so whole steps of
                                      // device-collective shards replay from a graph
  int hsent[2];                       // this step's boundary tiles pushed (low / high side)
  // CFL filter hint (k_speeds_b): per direction, the edge where the previous
  // step's max |s| was found, packed (speed bits >> 29) << 29 | edge index;
  // hint_acc[parity] accumulates this step's (64-bit MAX), the commit moves it
  unsigned long long hint_acc[2][2];
  unsigned long long hint[2];
  int tmax_ok[2];                     // tile maxima of state buffer p written by its update
  unsigned long long tnext[2][2];     // exact max|s| bits of one x / y edge of state buffer p
                                      // (the update that wrote it probed its hint edges)
  Report rep[REPCAP];
};

struct StepArgs {
  double dx, dy;
  double cfl, dt_max, fixed_dt, remaining, t_final, tol;
  int has_dt_max, has_fixed, has_remaining, has_t_final;
  int cur;              // slot parity of this step
  int static_speeds;    // 1: max speeds come from DevState::static_bits
  int* borders;         // tile-border counters of the fused CFL epilogue
  void* tmax;           // per-tile bound maxima [2][ntiles][4] R for k_speeds_t, or null
  int part;             // 0 whole step; 1 boundary tile rows; 2 interior tile rows
  int tr_lo, tr_hi;     // part 1 = tile rows [0, tr_lo) + [tr_hi, nty), part 2 = [tr_lo, tr_hi)
  int nblk_total;       // CTAs of the whole step over its parts (0: this grid)
};

__device__ __forceinline__ int map_i(int i, const Layout& L) {
  if (i < 0) i = (L.bcx == BC_PERIODIC) ? i + L.nx : 0;
  else if (i >= L.nx) i = (L.bcx == BC_PERIODIC) ? i - L.nx : L.nx - 1;
  // cells past the periodic image only feed discarded (out-of-domain) cells
  return i < 0 ? 0 : (i >= L.nx ? L.nx - 1 : i);
}

__device__ __forceinline__ int map_j(int j, const Layout& L) {
  if (j < 0) {
    if (L.lo == ROWS_MEMORY) return j < -2 ? -2 : j;
    j = (L.bcy == BC_PERIODIC) ? j + L.ny : 0;
  } else if (j >= L.ny) {
    if (L.hi == ROWS_MEMORY) return j > L.ny + 1 ? L.ny + 1 : j;
    j = (L.bcy == BC_PERIODIC) ? j - L.ny : L.ny - 1;
  }
  return j < 0 ? 0 : (j >= L.ny ? L.ny - 1 : j);
}

__device__ __forceinline__ long long row_off(int j, const Layout& L) {
  return (long long)(j + 2) * L.rstride;
}

// Error key: ordering of reference CellWise/Serial sweeps (sweep.py:203-218):
// all x chunks, then y; chunk = MAX_BLOCK // width rows (sweep.py:117-119);
// inside a chunk the kernel's admissibility stage, then the first bad element
// in C order over (component, i, j) (_first_bad, kernels.py:132-135).  63 bits, so the
// reduction slot stores NKEY_MAX - key >= 0 and one int64/u64 MAX all-reduce
// across shards picks the smallest key.
constexpr unsigned long long NKEY_MAX = 0x7fffffffffffffffull;
__device__ __forceinline__ unsigned long long err_key(int dir, int i, int jg, int stage,
                                                      int comp, int nx) {
  int width = dir == 0 ? nx + 1 : nx;
  int rows_per = 32768 / width;
  if (rows_per < 1) rows_per = 1;
  unsigned long long chunk = (unsigned long long)(jg / rows_per);
  return ((unsigned long long)dir << 62) | (chunk << 44) |
         ((unsigned long long)stage << 40) | ((unsigned long long)comp << 37) |
         ((unsigned long long)i << 18) | (unsigned long long)jg;
}

template <class R> struct Bits;
template <> struct Bits<double> {
  static __device__ __forceinline__ unsigned long long to(double v) {
    return (unsigned long long)__double_as_longlong(v);
  }
  static __device__ __forceinline__ double from(unsigned long long b) {
    return __longlong_as_double((long long)b);
  }
};
template <> struct Bits<float> {
  static __device__ __forceinline__ unsigned long long to(float v) {
    return (unsigned long long)__float_as_uint(v);
  }
  static __device__ __forceinline__ float from(unsigned long long b) {
    return __uint_as_float((unsigned)b);
  }
};

// numpy.minimum / maximum for non-NaN operands
template <class R> __device__ __forceinline__ R nmin(R a, R b) { return (a <= b) ? a : b; }
template <class R> __device__ __forceinline__ R nmax(R a, R b) { return (a >= b) ? a : b; }

// Step control computed identically by every CTA: dt from this step's max
// speeds exactly as reference choose_dt (driver.py:34-57), all in fp64.
struct Ctl {
  double dt, msx, msy;
  int skip;        // 1: do nothing (sticky error, pending error, or t_final reached)
  int stationary;  // rate == 0 without fixed_dt
  int finished;
};

template <class R>
__device__ __forceinline__ Ctl step_control(const StepArgs& A, const DevState* ds,
                                            bool pending_error_blocks) {
  Ctl c;
  c.skip = 0; c.stationary = 0; c.finished = 0; c.dt = 0.0;
  // plain L2 reads: everything read here was written by an earlier kernel
  // (the commit of the previous step / the speeds pre-pass)
  if (__ldcg(&ds->err)) { c.skip = 1; c.msx = c.msy = 0.0; return c; }
  unsigned long long bx, by;
  if (A.static_speeds) { bx = __ldcg(&ds->static_bits[0]); by = __ldcg(&ds->static_bits[1]); }
  else { bx = __ldcg(&ds->slot[A.cur][0]); by = __ldcg(&ds->slot[A.cur][1]); }
  c.msx = (double)Bits<R>::from(bx);
  c.msy = (double)Bits<R>::from(by);
  if (pending_error_blocks && __ldcg(&ds->slot[A.cur][2]) != 0ull) c.skip = 1;
  double remaining = A.remaining;
  int has_rem = A.has_remaining;
  if (A.has_t_final) {
    double t = __ldcg(&ds->t);
    if (!(A.t_final - t > A.tol)) { c.skip = 1; c.finished = 1; return c; }
    remaining = A.t_final - t;
    has_rem = 1;
  }
  double dt;
  if (A.has_fixed) {
    dt = A.fixed_dt;
  } else {
    double rate = c.msx / A.dx + c.msy / A.dy;
    if (rate == 0.0) { c.stationary = 1; c.skip = 1; return c; }
    dt = A.cfl / rate;
  }
  if (A.has_dt_max) dt = (A.dt_max < dt) ? A.dt_max : dt;   // Python min(dt, dt_max)
  if (has_rem) dt = (remaining < dt) ? remaining : dt;
  c.dt = dt;
  return c;
}

}  // namespace ws
