"""Device session: one C-ABI handle = one grid shard resident on one GPU.

``DeviceGrid`` is the native-facing object every higher layer uses
(driver.step/run, the row-strip orchestrator in parallel.py, bench.py).
It owns the handle, converts host arrays to the C ABI's expectations and
maps device error records to the reference's exception types
(SweepError / ValueError, reference sweep.py:68-75, driver.py:50-51).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _abi
from .kernels import DESCRIPTORS, STAGES, Direction, Kernel, KernelError
from .sweep import SweepError


@dataclass(frozen=True)
class Cuda:
    """Execution backend value for SimulationConfig (replaces Serial/StaticThreads/
    WorkStealing, reference parallel.py:39-74)."""

    device: int = 0
    precision: str = "f64"

    def __post_init__(self):
        if self.precision not in _abi.PRECISION_IDS:
            raise ValueError(f"precision must be one of {sorted(_abi.PRECISION_IDS)}")


@dataclass
class PollResult:
    steps_done: int
    reports: list          # list of (dt, cfl, max_speed_x, max_speed_y)
    t: float
    error: _abi.WsErrorInfo


STATIONARY_MSG = "all wave speeds are zero; a stationary field needs fixed_dt"


class DeviceGrid:
    """Device-resident grid shard with a bound solver."""

    def __init__(self, nx: int, ny: int, dx: float, dy: float, kernel: Kernel, *,
                 order: int = 1, limiter: str = "none", bc_x: str = "periodic",
                 bc_y: str = "periodic", precision: str = "f64", device: int = 0,
                 ny_global: int | None = None, j_offset: int = 0,
                 rows_lo: int = _abi.ROWS_BC, rows_hi: int = _abi.ROWS_BC,
                 buffers: dict | None = None):
        if limiter not in _abi.LIMITER_IDS:
            raise ValueError(f"unknown limiter {limiter!r}; choose from {sorted(_abi.LIMITER_IDS)}")
        if order not in (1, 2):
            raise ValueError(f"order must be 1 or 2, got {order}")
        self.lib = _abi.lib()
        self.kernel = kernel
        self.desc = DESCRIPTORS[kernel.name]
        self.nx, self.ny = int(nx), int(ny)
        self.precision = precision
        self.dtype = np.float64 if precision == "f64" else np.float32
        d = _abi.WsDesc()
        d.nx, d.ny, d.dx, d.dy = self.nx, self.ny, float(dx), float(dy)
        d.num_ghost = 2
        d.solver = _abi.SOLVER_IDS[kernel.name]
        for k, v in enumerate(kernel.native_params()):
            d.params[k] = float(v)
        d.order = order
        d.limiter = _abi.LIMITER_IDS[limiter]
        d.bc_x = _abi.BC_IDS[bc_x]
        d.bc_y = _abi.BC_IDS[bc_y]
        d.precision = _abi.PRECISION_IDS[precision]
        d.device = int(device)
        d.ny_global = int(ny if ny_global is None else ny_global)
        d.j_offset = int(j_offset)
        d.rows_lo, d.rows_hi = int(rows_lo), int(rows_hi)
        if buffers:
            d.ext_q0 = buffers.get("q0")
            d.ext_q1 = buffers.get("q1")
            d.ext_aux = buffers.get("aux")
            d.ext_slots = buffers.get("slots")
        self._desc = d
        h = ctypes.c_void_p()
        rc = self.lib.ws_create(ctypes.byref(d), ctypes.byref(h))
        if rc == _abi.WS_ERR_CONFIG:
            raise ValueError(self.lib.ws_last_error(None).decode())
        _abi.check(rc, None)
        self.h = h

    # -- lifecycle -----------------------------------------------------------
    def close(self):
        if getattr(self, "h", None):
            self.lib.ws_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc == _abi.WS_ERR_CONFIG:
            raise ValueError(self.lib.ws_last_error(self.h).decode())
        _abi.check(rc, self.h)

    # -- data movement ---------------------------------------------------------
    def host_shape(self, ncomp):
        return (ncomp, self.nx + 4, self.ny + 4)

    def _host(self, a, ncomp, name):
        if a.shape != self.host_shape(ncomp):
            raise ValueError(f"{name} must have shape {self.host_shape(ncomp)}, got {a.shape}")
        if a.dtype != self.dtype or not a.flags.f_contiguous:
            a = np.asfortranarray(a, dtype=self.dtype)
        return a

    def upload(self, q: np.ndarray, aux: np.ndarray | None = None, stream=None):
        q = self._host(q, self.desc.num_eqn, "state")
        ap = None
        if self.desc.num_aux:
            if aux is None:
                raise ValueError(f"{self.kernel.name} requires aux data")
            aux = self._host(aux, self.desc.num_aux, "aux")
            ap = aux.ctypes.data
        fn = self.lib.ws_upload if self.precision == "f64" else self.lib.ws_upload_f32
        self._check(fn(self.h, q.ctypes.data, ap, stream))

    def download(self, out: np.ndarray | None = None, stream=None, wait: bool = True
                 ) -> np.ndarray:
        """State with its ghost frame, host layout.  ``wait=False`` only
        enqueues the copy into ``out`` (ws_download_async): read it after the
        stream completes and ``poll`` shows no error."""
        shape = self.host_shape(self.desc.num_eqn)
        if not wait:
            if out is None or out.dtype != self.dtype or not out.flags.f_contiguous \
                    or out.shape != shape:
                raise ValueError(f"an async download needs a Fortran-ordered {shape} "
                                 f"{np.dtype(self.dtype).name} destination")
            self._check(self.lib.ws_download_async(self.h, out.ctypes.data, stream))
            return out
        buf = out if (out is not None and out.dtype == self.dtype and out.flags.f_contiguous
                      and out.shape == shape) else np.zeros(shape, dtype=self.dtype, order="F")
        fn = self.lib.ws_download if self.precision == "f64" else self.lib.ws_download_f32
        self._check(fn(self.h, buf.ctypes.data, stream))
        if out is not None and buf is not out:
            out[...] = buf
            return out
        return buf

    def download_aux_ghosts(self, aux: np.ndarray) -> np.ndarray:
        """Write the BC ghost frame of the uploaded aux into ``aux``'s ghost
        frame in place (ws_download_aux_ghosts; reference fill_ghost of aux
        in driver.py:211-212).  ``aux`` must be the handle's precision, F-order."""
        shape = self.host_shape(self.desc.num_aux)
        if aux.shape != shape or aux.dtype != self.dtype or not aux.flags.f_contiguous:
            raise ValueError(f"aux ghosts need a Fortran-ordered {shape} "
                             f"{np.dtype(self.dtype).name} array")
        self._check(self.lib.ws_download_aux_ghosts(self.h, aux.ctypes.data, None))
        return aux

    # -- stepping ---------------------------------------------------------------
    def step(self, ctl: _abi.WsCtl, stream=None):
        self._check(self.lib.ws_step(self.h, ctypes.byref(ctl), stream))

    def run(self, nsteps: int, ctl: _abi.WsCtl, stream=None):
        self._check(self.lib.ws_run(self.h, int(nsteps), ctypes.byref(ctl), stream))

    def phase_speeds(self, stream=None, part: int = 0):
        """CFL pre-pass; part 1/2 = before/after the low halo rows arrive
        (ws_phase_speeds_part), 0 = whole."""
        self._check(self.lib.ws_phase_speeds_part(self.h, int(part), stream))

    def phase_update(self, ctl: _abi.WsCtl, stream=None, part: int = 0):
        """Update; part 1/2 = boundary / interior tile rows of a shard
        (ws_phase_update_part), 0 = whole."""
        if part == 0:
            self._check(self.lib.ws_phase_update(self.h, ctypes.byref(ctl), stream))
        else:
            self._check(self.lib.ws_phase_update_part(self.h, ctypes.byref(ctl), int(part),
                                                      stream))

    def capture_begin(self):
        """Before the caller captures whole steps of phase calls into its own
        CUDA graph (ws_capture_begin)."""
        self._check(self.lib.ws_capture_begin(self.h))

    def capture_end(self) -> tuple[int, int]:
        """(steps, launches) the captured calls stand for; the handle's
        counts roll back, nothing ran (ws_capture_end)."""
        st, ln = ctypes.c_int64(), ctypes.c_int64()
        self._check(self.lib.ws_capture_end(self.h, ctypes.byref(st), ctypes.byref(ln)))
        return int(st.value), int(ln.value)

    def replayed(self, steps: int, launches: int):
        """After each replay of such a graph (ws_replayed)."""
        self._check(self.lib.ws_replayed(self.h, int(steps), int(launches)))

    def slot_ptr(self) -> int:
        return self.lib.ws_slot_ptr(self.h)

    def halo_ptrs(self):
        p = [ctypes.c_void_p() for _ in range(4)]
        nb = ctypes.c_uint64()
        self._check(self.lib.ws_halo_ptrs(self.h, *[ctypes.byref(x) for x in p],
                                          ctypes.byref(nb)))
        return [x.value for x in p], nb.value

    def state_ptr(self):
        q = ctypes.c_void_p()
        pitch = ctypes.c_int64()
        row = ctypes.c_int64()
        self._check(self.lib.ws_state_ptr(self.h, ctypes.byref(q), ctypes.byref(pitch),
                                          ctypes.byref(row)))
        return q.value, pitch.value, row.value

    def sync(self):
        self._check(self.lib.ws_sync(self.h))

    def devstate_ptr(self) -> int:
        return self.lib.ws_devstate_ptr(self.h)

    def set_halo_peers(self, lo=None, hi=None):
        """Device-side halo push (ws_set_halo_peers): lo = (q0, q1, state,
        ny) of the low neighbour, hi = (q0, q1, state) of the high one, as
        device pointers mapped on this GPU; None = no neighbour."""
        lq = (ctypes.c_void_p * 2)(*(lo[:2] if lo else (None, None)))
        hq = (ctypes.c_void_p * 2)(*(hi[:2] if hi else (None, None)))
        self._check(self.lib.ws_set_halo_peers(self.h, lq, lo[2] if lo else None,
                                               int(lo[3]) if lo else 0, hq,
                                               hi[2] if hi else None))

    def set_peers(self, state_ptrs):
        """Device-side CFL reduction across shards (ws_set_peers): the
        DevState pointers of every shard as mapped on this GPU, self
        included; [] turns it off."""
        arr = (ctypes.c_void_p * max(1, len(state_ptrs)))(*state_ptrs)
        self._check(self.lib.ws_set_peers(self.h, len(state_ptrs), arr))

    def checked_counts(self):
        """Checked builds (WAVESTEP_LIB=_lib/checked/libwavestep.so): (violation
        bits, min, max of the per-cell write counts) since the upload."""
        f, lo, hi = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        self._check(self.lib.ws_checked_counts(self.h, ctypes.byref(f), ctypes.byref(lo),
                                               ctypes.byref(hi)))
        return f.value, lo.value, hi.value

    def launches(self) -> int:
        return int(self.lib.ws_launch_count(self.h))

    def poll(self, max_reports: int = 4096) -> PollResult:
        steps = ctypes.c_int64()
        reps = (_abi.WsReport * max_reports)()
        nrep = ctypes.c_int32()
        t = ctypes.c_double()
        err = _abi.WsErrorInfo()
        rc = self.lib.ws_poll(self.h, ctypes.byref(steps), reps, max_reports,
                              ctypes.byref(nrep), ctypes.byref(t), ctypes.byref(err))
        if rc not in (_abi.WS_OK, _abi.WS_ERR_KERNEL, _abi.WS_ERR_STATIONARY):
            self._check(rc)
        out = [(r.dt, r.cfl, r.max_speed_x, r.max_speed_y) for r in reps[:nrep.value]]
        return PollResult(int(steps.value), out, float(t.value), err)

    def raise_for(self, err: _abi.WsErrorInfo):
        """Re-raise a device error record as the reference's exception."""
        if err.code == _abi.WS_ERR_KERNEL:
            reason, side = STAGES[self.kernel.name][err.stage]
            direction = Direction.X if err.direction == 0 else Direction.Y
            raise SweepError(direction, err.i, err.j, KernelError(reason, side=side))
        if err.code == _abi.WS_ERR_STATIONARY:
            raise ValueError(STATIONARY_MSG)
        if err.code:
            raise _abi.NativeError(err.code, f"device error {err.code}")
