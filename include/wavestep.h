/*
 * wavestep.h — C ABI of the B200-native 2D wave-propagation step.
 *
 * Drop-in boundary for the hot path of the reference package `wavesweep`
 * (/root/reference/pkg/src/wavesweep).  The reference is pure Python, so
 * its "FFI" is the Python call surface; each entry point below states the
 * reference interface it replaces.  The Python host layer
 * (paper_1308_1464_b200/_abi.py) binds exactly these symbols with ctypes;
 * INTEGRATION.md shows the binding.
 *
 * Types are plain C: no torch or CUDA types appear in the signatures
 * (streams are passed as `void*` holding a cudaStream_t, NULL = the
 * handle's own stream).  All reals on the host side are float64 in the
 * reference's layout: arrays of shape (ncomp, nx+4, ny+4), Fortran order
 * (component fastest, then i, then j), two ghost layers
 * (reference grid.py:76-95).  Device storage is the handle's own
 * structure-of-arrays layout.
 *
 * Return codes (every int-returning function):
 *   WS_OK (0), WS_ERR_KERNEL (1: inadmissible state, see ws_error_info),
 *   WS_ERR_CONFIG (2: bad descriptor / argument, message in ws_last_error),
 *   WS_ERR_CUDA (3), WS_ERR_STATIONARY (4: all wave speeds zero and no
 *   fixed_dt — reference driver.py:50-51 raises ValueError), WS_ERR_INTERNAL
 *   (5: a device-side invariant check failed -- a bug, never the input).
 */
#ifndef WAVESTEP_H
#define WAVESTEP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WS_ABI_VERSION 1

enum ws_status { WS_OK = 0, WS_ERR_KERNEL = 1, WS_ERR_CONFIG = 2, WS_ERR_CUDA = 3,
                 WS_ERR_STATIONARY = 4, WS_ERR_INTERNAL = 5 };

/* Riemann solvers: reference kernels.py:89-94 (DESCRIPTORS) plus the two
 * north-star solvers the reference lacks. */
enum ws_solver { WS_ACOUSTICS_CONST = 0,   /* kernels.py:181-213, params rho, bulk      */
                 WS_ACOUSTICS_VAR = 1,     /* kernels.py:216-261, aux (rho, c) rp_acoustics_var */
                 WS_EULER_ROE = 2,         /* kernels.py:264-340, params gamma          */
                 WS_EULER_HLLE = 3,        /* extension, params gamma                   */
                 WS_SHALLOW_ROE = 4,       /* extension (Roe + Harten fix), params grav */
                 WS_ADVECTION = 5 };       /* kernels.py:163-178, rp_advection u, v   */

enum ws_limiter { WS_LIM_NONE = 0, WS_LIM_MINMOD = 1, WS_LIM_SUPERBEE = 2, WS_LIM_MC = 3 };
enum ws_bc { WS_BC_PERIODIC = 0, WS_BC_EXTRAPOLATE = 1 };  /* grid.py:12-16 */
/* WS_FP32: the fp32 step bitwise equal to a float32 run of the oracle (no
 * FMA contraction, IEEE division / square root).  WS_FP32_FAST: the fp32
 * throughput mode -- FMA contraction, the approximate MUFU division /
 * square root, denormals flushed to zero; its parity is the stated bound
 * against fp64 (max relative error <= 1e-5 on the state and on every dt
 * after 20 steps), not bits. */
enum ws_precision { WS_FP64 = 0, WS_FP32 = 1, WS_FP32_FAST = 2 };
/* how the rows below j = 0 / above j = ny of THIS shard are obtained */
enum ws_rowmode { WS_ROWS_MEMORY = 0,   /* ghost rows in memory (halo exchange) */
                  WS_ROWS_BC = 1 };     /* physical boundary: apply bc_y         */

/* Replaces GridSpec (grid.py:19-50) + SimulationConfig (driver.py:60-83)
 * + make_kernel (kernels.py:396-440) for one shard. */
typedef struct ws_desc {
  int32_t nx, ny;            /* interior cells of this shard (ny = local rows)      */
  double dx, dy;             /* cell widths                                         */
  int32_t num_ghost;         /* must be 2 (reference default grid.py:36)            */
  int32_t solver;            /* enum ws_solver                                      */
  double params[4];          /* acoustics-const: rho, bulk; euler*: gamma; sw: grav;
                                advection: u, v                                      */
  int32_t order;             /* 1 = reference donor cell, 2 = + limited correction */
  int32_t limiter;           /* enum ws_limiter (ignored for order 1)               */
  int32_t bc_x, bc_y;        /* enum ws_bc                                          */
  int32_t precision;         /* enum ws_precision                                   */
  int32_t device;            /* CUDA ordinal                                        */
  /* row-strip decomposition (reference has none: SPEC.md:89 non-goal) */
  int32_t ny_global;         /* rows of the whole domain (== ny for one shard)      */
  int32_t j_offset;          /* global row of local row 0                            */
  int32_t rows_lo, rows_hi;  /* enum ws_rowmode for the bottom / top ghost rows     */
  /* optional borrowed device buffers (NULL = the handle allocates).  Sizes
   * from ws_buffer_bytes().  q0 receives uploads; steps ping-pong q0 <-> q1. */
  void *ext_q0, *ext_q1, *ext_aux, *ext_slots;
} ws_desc;

/* Replaces TimestepController (driver.py:17-31) + the `remaining`
 * argument of step() (driver.py:199-201).  NaN = "None". */
typedef struct ws_ctl {
  double cfl;        /* cfl_target in (0,1)                   */
  double dt_max;     /* NaN = None                            */
  double fixed_dt;   /* NaN = None                            */
  double remaining;  /* NaN = None (per-step clamp)           */
  double t_final;    /* NaN = None; device-side run() target  */
} ws_ctl;

/* Replaces StepReport (driver.py:86-95), minus the wall-clock fields. */
typedef struct ws_report {
  double dt, cfl, max_speed_x, max_speed_y;
} ws_report;

/* Replaces SweepError (sweep.py:68-75) / KernelError (kernels.py:44-55). */
typedef struct ws_error_info {
  int32_t code;        /* 0 none, else enum ws_status                          */
  int32_t direction;   /* 0 = x-interface, 1 = y-interface                     */
  int32_t i, j;        /* global interface indices                              */
  int32_t stage;       /* index of the failed admissibility test, solver order  */
  int32_t component;   /* component for non-finite tests                        */
  int64_t step;        /* step index (since upload) that failed                */
} ws_error_info;

typedef struct ws_handle ws_handle;

int ws_abi_version(void);

/* Layout of the borrowed buffers a caller may provide in ws_desc. */
int ws_buffer_bytes(const ws_desc* d, uint64_t* q_bytes, uint64_t* aux_bytes,
                    uint64_t* slots_bytes);

int ws_create(const ws_desc* d, ws_handle** out);
void ws_destroy(ws_handle* h);
/* last message; h may be NULL for ws_create failures */
const char* ws_last_error(const ws_handle* h);

/* Host <-> device.  Host arrays use the reference layout (ncomp, nx+4, ny+4)
 * Fortran order.  Pinned host memory makes the copies asynchronous.
 * Replaces the StateField/AuxField data hand-off (grid.py:86-95). */
int ws_upload(ws_handle* h, const double* q_host, const double* aux_host, void* stream);
int ws_download(ws_handle* h, double* q_host, void* stream);
/* fp32 handles: same calls with float arrays */
int ws_upload_f32(ws_handle* h, const float* q_host, const float* aux_host, void* stream);
int ws_download_f32(ws_handle* h, float* q_host, void* stream);
/* Enqueue-only download (array of the handle's precision): no host sync and
 * no device error check — valid after the stream completes and ws_poll
 * reports no error.  With a pinned destination it overlaps the next
 * ws_upload's host-to-device copy issued on another stream.
 *
 * Streams: a null stream selects the handle's own stream.  Operations on one
 * handle execute in issue order whatever streams they are issued on (a call
 * on a different stream than the previous one waits for it), with two
 * relaxations that let transfers overlap: ws_upload's host-to-device copy
 * may start before earlier work finishes (it runs on the handle's copy stream
 * into one of two alternating staging buffers; the conversion into the
 * state, on the caller's stream, waits for it, so the host array may be
 * reused once the caller's stream has passed the upload), and work issued after a download
 * on another stream does not wait for that download's device-to-host copy
 * (wait for the stream, or use the synchronous ws_download, before reading
 * the host array). */
int ws_download_async(ws_handle* h, void* q_host, void* stream);

/* The BC ghost frame of the aux the last ws_upload carried, filled like the
 * reference's fill_ghost (grid.py:179-193) from its interior, written into
 * the ghost frame of the host aux array (reference layout); the interior is
 * left untouched.  The reference's step refills the caller's aux ghosts
 * every step (driver.py:211-212); this is that mutation.  Synchronous.
 * No-op for solvers without aux. */
int ws_download_aux_ghosts(ws_handle* h, void* aux_host, void* stream);

/* Page-lock (cudaHostRegister, portable) / release a caller's host array so
 * ws_upload / ws_download copy it by DMA at full PCIe rate.  The drop-in
 * driver.step pins the caller's StateField / AuxField arrays once per array
 * (the reference's step mutates them in place, driver.py:199-225). */
int ws_pin_host(void* ptr, uint64_t bytes);
int ws_unpin_host(void* ptr);

/* Checked builds only (-DWS_CHECKED=1; the device analogue of the
 * reference's WAVESWEEP_CHECKED write counts, sweep.py:32-33, 78-96): the
 * bits of every device index check that failed since the last upload, and
 * the minimum / maximum over the interior cells of the update kernel's
 * write counts (each step writes every cell exactly once).  Other builds
 * return WS_ERR_CONFIG. */
int ws_checked_counts(ws_handle* h, uint32_t* flags, uint32_t* writes_min, uint32_t* writes_max);

/* One step, enqueued only (no host sync): fill ghosts (implicit, by index
 * mapping) -> sweep -> choose_dt on device -> update.
 * Replaces driver.step (driver.py:199-225). */
int ws_step(ws_handle* h, const ws_ctl* c, void* stream);
/* nsteps steps through a captured CUDA graph; stops early on error or when
 * t_final is reached.  Replaces driver.run's loop (driver.py:228-250). */
int ws_run(ws_handle* h, int32_t nsteps, const ws_ctl* c, void* stream);

/* Split step for multi-shard runs: the caller all-reduces the 3 x uint64
 * slot (MAX) between the two phases and exchanges halo rows before phase 1.
 * ws_step == ws_phase_speeds + ws_phase_update on one shard. */
int ws_phase_speeds(ws_handle* h, void* stream);
/* ws_phase_speeds in two parts, so a shard overlaps the pre-pass with its
 * halo exchange: part 1 = every edge except the y-edges that read received
 * ghost rows (local row 0, and row ny of a top shard whose high ghost rows
 * come from a periodic neighbour), enqueued while the halo rows are in
 * flight; part 2 = those y-edges, after they arrived.  part 0 = both. */
int ws_phase_speeds_part(ws_handle* h, int32_t part, void* stream);
int ws_phase_update(ws_handle* h, const ws_ctl* c, void* stream);
/* ws_phase_update in two launches so a shard overlaps its halo exchange with
 * the update: part 1 = the tile rows holding local rows 0, 1 and ny-2, ny-1
 * (the rows the neighbours need as ghost rows of the next step), part 2 =
 * the interior tile rows; the caller sends the new boundary rows after part
 * 1 while part 2 runs.  Call part 1 then part 2 with the same control; the
 * step counts as done after part 2.  part 0 == ws_phase_update. */
int ws_phase_update_part(ws_handle* h, const ws_ctl* c, int32_t part, void* stream);
/* Caller-side graph capture of whole steps of phase calls (a torch CUDA
 * graph that also holds the NCCL slot all-reduce and halo send/recv): call
 * ws_capture_begin before capturing the phase calls and ws_capture_end after
 * it; it returns the steps (must be even: the ping-pong parity repeats) and
 * kernel launches the captured calls stand for, and rolls this handle's
 * step and launch counts back, since nothing ran.  After each replay of the
 * graph, ws_replayed(h, steps, launches) advances them as the calls would
 * have.  Not a reference interface: the reference steps from Python. */
int ws_capture_begin(ws_handle* h);
int ws_capture_end(ws_handle* h, int64_t* steps, int64_t* launches);
int ws_replayed(ws_handle* h, int64_t steps, int64_t launches);
/* device pointer of the current step's 3 x uint64 reduction slot */
void* ws_slot_ptr(ws_handle* h);
/* device pointers of the current state's halo rows (2 rows x all components,
 * contiguous): send_lo = rows 0,1; send_hi = rows ny-2,ny-1; recv_lo = rows
 * -2,-1; recv_hi = rows ny,ny+1.  bytes = size of each block. */
int ws_halo_ptrs(ws_handle* h, void** send_lo, void** send_hi, void** recv_lo,
                 void** recv_hi, uint64_t* bytes);
/* device pointer of the current state buffer and its row geometry */
int ws_state_ptr(ws_handle* h, void** q, int64_t* pitch_elems, int64_t* row_elems);

/* Synchronise and read what the device recorded: number of committed steps
 * since upload, their reports (the last min(n, max) of them), time t, and
 * the error record.  Reports are consumed (cleared) by this call. */
int ws_poll(ws_handle* h, int64_t* steps_done, ws_report* reports, int32_t max_reports,
            int32_t* n_reports, double* t_now, ws_error_info* err);
int ws_sync(ws_handle* h);

/* Pointwise plugin call, batched: replaces Kernel.solve(direction, ql, qr,
 * auxl, auxr) -> RiemannResult (kernels.py:374-393) for one solver on n
 * interfaces.  Host arrays, C order: ql/qr (num_eqn, n), aux (num_aux, n)
 * or NULL, waves (num_waves, num_eqn, n), speeds (num_waves, n),
 * amdq/apdq (num_eqn, n), codes (n): 0 admissible, else
 * (stage + 1) | (component << 8) of the first failed test in the
 * reference's order.  direction 0 = x, 1 = y.  fp64 only. */
int ws_riemann(int32_t solver, const double* params, int32_t direction, int64_t n,
               const double* ql, const double* qr, const double* auxl, const double* auxr,
               double* waves, double* speeds, double* amdq, double* apdq, int32_t* codes,
               int32_t device);

/* In-place ghost fill of a host field (ncomp, nx+4, ny+4) F-order on the
 * device: replaces fill_ghost (grid.py:179-193; x pass then y pass). */
int ws_fill_ghost(double* data, int32_t ncomp, int32_t nx, int32_t ny, int32_t bc_x,
                  int32_t bc_y, int32_t device);

/* number of kernel launches this handle has issued (bench evidence) */
int64_t ws_launch_count(const ws_handle* h);

/* Device-side CFL reduction across row-strip shards (replaces the host
 * all-reduce of the slot between ws_phase_speeds and ws_phase_update): with
 * npeers > 0, the last CTA of each pre-pass (part 0 or 2) max-reduces this
 * shard's 3-word slot into every table entry's slot (64-bit system-scope
 * atomics; peers reached through P2P / symmetric-memory mappings) and
 * increments their arrival counters; the update waits until npeers pushes
 * for the step arrived.  peer_states[r] = ws_devstate_ptr of shard r as
 * mapped on this GPU (self included); npeers = 0 turns it off.  All shards
 * must ws_upload before any shard steps. */
#define WS_MAX_PEERS 8
int ws_set_peers(ws_handle* h, int32_t npeers, void* const* peer_states);
void* ws_devstate_ptr(ws_handle* h);
/* Device-side halo exchange (replaces the host halo send/recv): the update
 * kernel stores this shard's two first / last rows straight into the low /
 * high neighbour's ghost rows (lo_q / hi_q = the neighbour's two state
 * buffers, ping-pong order, as mapped on this GPU; ny_lo = the low
 * neighbour's row count) and releases the neighbour's arrival counter
 * (lo_state / hi_state = its DevState); the pre-pass (part 2 / 0) waits for
 * the pushes it is owed before reading ghost rows.  Null state = that side
 * has no neighbour.  Use with ws_set_peers (the slot reduction orders the
 * buffer reuse across shards). */
int ws_set_halo_peers(ws_handle* h, void* const* lo_q, void* lo_state, int32_t ny_lo,
                      void* const* hi_q, void* hi_state);

/* Diagnostics (no reference counterpart): with WS_TRACE=1 in the environment
 * at ws_create, every CTA of the CFL pre-pass (region 0) and of the update
 * kernel (region 1) writes {start ns, end ns, smid, block} (%globaltimer) on
 * each launch.  Copies up to `cap` words of the last launch's records;
 * *n = 0 when tracing is off. */
int ws_trace(ws_handle* h, uint64_t* out, int64_t cap, int64_t* n);

#ifdef __cplusplus
}
#endif

#endif /* WAVESTEP_H */
