"""Riemann-solver plugins of the drop-in API (reference kernels.py).

The physics lives in CUDA device-function templates (csrc/ws_solvers.cuh)
that know nothing of tiles or threads.  This module is their host-side
registry: descriptors, parameter binding (``make_kernel``) and
``Kernel.solve`` — the reference's batched pointwise plugin call
(kernels.py:374-393) — executed on the GPU through ``ws_riemann``.
"""

from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _abi

ADMISSIBILITY_FLOOR = 1e-300  # reference kernels.py:34


class Direction(enum.Enum):
    X = "x"
    Y = "y"


class KernelError(ValueError):
    """Inadmissible kernel input (reference kernels.py:44-55)."""

    def __init__(self, message: str, side: str | None = None, element: tuple | None = None):
        super().__init__(message)
        self.side = side
        self.element = element


@dataclass(frozen=True)
class RiemannResult:
    waves: np.ndarray    # (num_waves, num_eqn) + batch
    speeds: np.ndarray   # (num_waves,) + batch
    amdq: np.ndarray     # (num_eqn,) + batch
    apdq: np.ndarray     # (num_eqn,) + batch


@dataclass(frozen=True)
class KernelDescriptor:
    name: str
    num_eqn: int
    num_waves: int
    num_aux: int
    arithmetic_intensity: Fraction


# reference kernels.py:89-94 plus the two north-star solvers the reference lacks
DESCRIPTORS: dict[str, KernelDescriptor] = {
    "advection": KernelDescriptor("advection", 1, 1, 0, Fraction(1, 3)),
    "acoustics-const": KernelDescriptor("acoustics-const", 3, 2, 0, Fraction(4, 5)),
    "acoustics-var": KernelDescriptor("acoustics-var", 3, 2, 2, Fraction(1)),
    "euler": KernelDescriptor("euler", 4, 3, 0, Fraction(1)),
    "euler-hlle": KernelDescriptor("euler-hlle", 4, 2, 0, Fraction(1)),
    "shallow-water-roe": KernelDescriptor("shallow-water-roe", 3, 3, 0, Fraction(1)),
}
KERNEL_NAMES = tuple(DESCRIPTORS)

# reason text per admissibility stage, in the order the device tests them
# (reference _check_states / _check_positive, kernels.py:145-156, 235-237, 280-301)
_FINITE = [("non-finite left state", "left"), ("non-finite right state", "right")]
STAGES = {
    "advection": _FINITE,
    "acoustics-const": _FINITE,
    "acoustics-var": _FINITE + [("nonpositive density on left side", "left"),
                                ("nonpositive sound speed on left side", "left"),
                                ("nonpositive density on right side", "right"),
                                ("nonpositive sound speed on right side", "right")],
    "euler": _FINITE + [("nonpositive density on left side", "left"),
                        ("nonpositive density on right side", "right"),
                        ("nonpositive pressure on left side", "left"),
                        ("nonpositive pressure on right side", "right"),
                        ("Roe-average sound speed is not real", None)],
    "shallow-water-roe": _FINITE + [("nonpositive depth on left side", "left"),
                                    ("nonpositive depth on right side", "right")],
}
STAGES["euler-hlle"] = STAGES["euler"]


@dataclass(frozen=True)
class AcousticsParams:
    density: float
    bulk: float

    def __post_init__(self):
        if not (self.density > 0 and self.bulk > 0):
            raise ValueError(f"density and bulk modulus must be positive, got "
                             f"{self.density}, {self.bulk}")

    @property
    def sound_speed(self) -> float:
        return math.sqrt(self.bulk / self.density)

    @property
    def impedance(self) -> float:
        return self.density * self.sound_speed


@dataclass(frozen=True)
class EulerParams:
    gamma: float = 1.4

    def __post_init__(self):
        if not self.gamma > 1.0:
            raise ValueError(f"gamma must exceed 1, got {self.gamma}")


@dataclass(frozen=True)
class ShallowWaterParams:
    grav: float = 9.81

    def __post_init__(self):
        if not self.grav > 0.0:
            raise ValueError(f"gravity must be positive, got {self.grav}")


class Kernel:
    """A solver bound to parameters; ``solve`` runs it on the GPU."""

    def __init__(self, descriptor: KernelDescriptor, params: dict):
        self.descriptor = descriptor
        self.params = dict(params)

    @property
    def name(self) -> str:
        return self.descriptor.name

    def native_params(self) -> list[float]:
        p = self.params
        if self.name == "advection":
            return [p["u"], p["v"], 0.0, 0.0]
        if self.name == "acoustics-const":
            return [p["rho"], p["bulk"], 0.0, 0.0]
        if self.name in ("euler", "euler-hlle"):
            return [p["gamma"], 0.0, 0.0, 0.0]
        if self.name == "shallow-water-roe":
            return [p["grav"], 0.0, 0.0, 0.0]
        return [0.0] * 4

    def __repr__(self):
        args = ", ".join(f"{k}={v}" for k, v in self.params.items())
        return f"Kernel({self.name}, {args})"

    def solve(self, direction: Direction, ql, qr, auxl=None, auxr=None) -> RiemannResult:
        """Batched pointwise solve (reference Kernel.solve / rp_*), on the device.

        Raises KernelError for the first inadmissible interface in the
        reference's order (stage, then C order over (component, batch)).
        """
        d = self.descriptor
        ql = np.asarray(ql, dtype=np.float64)
        qr = np.asarray(qr, dtype=np.float64)
        if ql.shape != qr.shape or ql.ndim < 1 or ql.shape[0] != d.num_eqn:
            raise ValueError(f"states must share a ({d.num_eqn}, ...) shape, got "
                             f"{ql.shape} and {qr.shape}")
        batch = ql.shape[1:]
        n = int(np.prod(batch)) if batch else 1
        a = np.ascontiguousarray(ql.reshape(d.num_eqn, n))
        b = np.ascontiguousarray(qr.reshape(d.num_eqn, n))
        al = ar = None
        if d.num_aux:
            if auxl is None or auxr is None:
                raise ValueError(f"{self.name} requires aux data on both sides")
            auxl = np.asarray(auxl, dtype=np.float64)
            auxr = np.asarray(auxr, dtype=np.float64)
            if auxl.shape != (d.num_aux,) + batch or auxr.shape != (d.num_aux,) + batch:
                raise ValueError(f"aux must have shape ({d.num_aux}, ...) matching the "
                                 f"states, got {auxl.shape}, {auxr.shape}")
            al = np.ascontiguousarray(auxl.reshape(d.num_aux, n))
            ar = np.ascontiguousarray(auxr.reshape(d.num_aux, n))
        waves = np.empty((d.num_waves, d.num_eqn, n))
        speeds = np.empty((d.num_waves, n))
        amdq = np.empty((d.num_eqn, n))
        apdq = np.empty((d.num_eqn, n))
        codes = np.empty(n, dtype=np.int32)
        prm = np.array(self.native_params(), dtype=np.float64)
        lib = _abi.lib()
        rc = lib.ws_riemann(
            _abi.SOLVER_IDS[self.name],
            prm.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            0 if Direction(direction) is Direction.X else 1, n,
            a.ctypes.data, b.ctypes.data,
            al.ctypes.data if al is not None else None,
            ar.ctypes.data if ar is not None else None,
            waves.ctypes.data, speeds.ctypes.data, amdq.ctypes.data, apdq.ctypes.data,
            codes.ctypes.data, 0)
        _abi.check(rc)
        bad = np.nonzero(codes)[0]
        if bad.size:
            stage = (codes[bad] & 0xFF) - 1
            comp = codes[bad] >> 8
            order = np.lexsort((bad, comp, stage))
            k = bad[order[0]]
            reason, side = STAGES[self.name][(codes[k] & 0xFF) - 1]
            element = tuple(int(x) for x in np.unravel_index(k, batch)) if batch else ()
            raise KernelError(reason, side=side, element=element)
        return RiemannResult(waves.reshape((d.num_waves, d.num_eqn) + batch),
                             speeds.reshape((d.num_waves,) + batch),
                             amdq.reshape((d.num_eqn,) + batch),
                             apdq.reshape((d.num_eqn,) + batch))


def make_kernel(name: str, **params) -> Kernel:
    """Bind a solver to parameters (reference kernels.py:396-440).

    advection(u, v), acoustics-const(rho, bulk), acoustics-var() reading per-cell (rho, c)
    from aux, euler(gamma=1.4), euler-hlle(gamma=1.4),
    shallow-water-roe(grav=9.81).
    """
    if name == "advection":
        u, v = float(params.pop("u")), float(params.pop("v"))
        if not (math.isfinite(u) and math.isfinite(v)):
            raise KernelError(f"non-finite advection velocity ({u}, {v})")
        bound = {"u": u, "v": v}
    elif name == "acoustics-const":
        p = AcousticsParams(float(params.pop("rho")), float(params.pop("bulk")))
        bound = {"rho": p.density, "bulk": p.bulk}
    elif name == "acoustics-var":
        bound = {}
    elif name in ("euler", "euler-hlle"):
        bound = {"gamma": EulerParams(float(params.pop("gamma", 1.4))).gamma}
    elif name == "shallow-water-roe":
        bound = {"grav": ShallowWaterParams(float(params.pop("grav", 9.81))).grav}
    else:
        raise ValueError(f"unknown kernel {name!r}; available: {', '.join(KERNEL_NAMES)}")
    if params:
        raise ValueError(f"unexpected parameters for {name}: {sorted(params)}")
    return Kernel(DESCRIPTORS[name], bound)
