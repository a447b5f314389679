"""CPU oracle for the 2D wave-propagation step — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` / ``--impl reference``) may import this module, and only
as the checker or as the timed CPU baseline.  The product package
(``paper_1308_1464_b200``) never imports it and has no CPU fallback.

What it restates
----------------
A numpy restatement of the reference's hot path
(``/root/reference/pkg/src/wavesweep``, "the reference" below):

* ghost fill ........ grid.py:156-193 (x pass over the full y extent, then y)
* Riemann kernels ... kernels.py:181-261 (acoustics const/var),
                      kernels.py:264-340 (Euler Roe, no entropy fix)
* admissibility ..... kernels.py:138-156 (finite first, then positivity,
                      left before right), ADMISSIBILITY_FLOOR 1e-300 (kernels.py:34)
* sweep ............. sweep.py:111-163 (x-edge i between cells i-1,i for
                      j in [0,ny); y-edge j between rows j-1,j for i in
                      [0,nx)); max |s| over exactly that edge set
* error location .... _locate, sweep.py:166-168, 203-243 (CellWise/Serial order:
                      all x chunks of MAX_BLOCK//width rows, then y)
* choose_dt ......... driver.py:34-57
* donor-cell update . sweep.py:254-280 (x term then y term, fixed order)
* step / run ........ driver.py:199-250

Every arithmetic expression keeps numpy's left-to-right association of the
reference so that ``order=1`` is BITWISE identical to ``wavesweep.driver.step``
(pinned by tests/test_oracle_pin.py against the live reference and against
tests/golden/*.npz generated from it).

Extension (not in the reference; "parity unpinned" by any reference test —
anchored instead by order-1 reduction, the Roe/conservation property,
X/Y symmetry, conservation and the exact Sod solution):

* shallow-water Roe solver with Harten's entropy fix (LeVeque 2002 §15.3)
* Euler HLLE solver (Einfeldt 1988, Roe-averaged bounds)
* wave limiters minmod / superbee / MC and the second-order correction flux
  (LeVeque 1997 wave propagation; no transverse terms)

The CUDA kernels in ``paper_1308_1464_b200/csrc`` evaluate the very same
expressions in the same order (compiled with ``--fmad=false``), which is
what makes fp64 parity bitwise rather than merely close.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

FLOOR = 1e-300          # reference kernels.py:34 (ADMISSIBILITY_FLOOR)
MAX_BLOCK = 1 << 15     # reference _MAX_BLOCK, sweep.py:30 — only used to order errors
PERIODIC = "periodic"
EXTRAPOLATE = "extrapolate"
LIMITERS = ("none", "minmod", "superbee", "mc")


class OracleError(ValueError):
    """First inadmissible edge, located like reference sweep.py:68-75."""

    def __init__(self, direction: str, i: int, j: int, reason: str, side):
        super().__init__(f"{direction}-interface (i={i}, j={j}): {reason}")
        self.direction, self.i, self.j = direction, i, j
        self.reason, self.side = reason, side


# ---------------------------------------------------------------------------
# grid: (ncomp, nx+2g, ny+2g) Fortran-ordered arrays like reference grid.py:89


def new_field(ncomp: int, nx: int, ny: int, g: int = 2) -> np.ndarray:
    return np.zeros((ncomp, nx + 2 * g, ny + 2 * g), order="F")


def interior(a: np.ndarray, g: int = 2) -> np.ndarray:
    return a[:, g:a.shape[1] - g, g:a.shape[2] - g]


def _fill(a: np.ndarray, n: int, g: int, bc: str, axis: int):
    # reference grid.py:156-176
    def s(lo, hi):
        idx = [slice(None)] * a.ndim
        idx[axis] = slice(lo, hi)
        return tuple(idx)

    if bc == PERIODIC:
        if n < g:
            raise ValueError(f"periodic boundary needs at least num_ghost={g} "
                             f"interior cells, got {n}")
        a[s(0, g)] = a[s(n, n + g)]
        a[s(g + n, 2 * g + n)] = a[s(g, 2 * g)]
    elif bc == EXTRAPOLATE:
        a[s(0, g)] = a[s(g, g + 1)]
        a[s(g + n, 2 * g + n)] = a[s(g + n - 1, g + n)]
    else:
        raise ValueError(f"unknown boundary condition {bc!r}")


def fill_ghost(a: np.ndarray, bc_x: str, bc_y: str, g: int = 2):
    """x pass over the full y extent, then the y pass (grid.py:179-193)."""
    if a.shape[0] == 0:
        return a
    nx, ny = a.shape[1] - 2 * g, a.shape[2] - 2 * g
    _fill(a, nx, g, bc_x, 1)
    _fill(a, ny, g, bc_y, 2)
    return a


# ---------------------------------------------------------------------------
# Riemann solvers.  Each takes the normal slot ni (1 = x, 2 = y), left/right
# states of shape (neq, ...) and aux (naux, ...), and returns
# (waves (mw, neq, ...), speeds (mw, ...), amdq (neq, ...), apdq (neq, ...)).
# `checks` lists the admissibility tests in the reference's order:
# (reason, side, bad-mask[, per-component]).


def _finite_checks(ql, qr):
    # kernels.py:145-148: left then right; element = first bad in C order
    # over (component, batch...) — i.e. the lowest component wins
    return [("non-finite left state", "left", ~np.isfinite(ql), True),
            ("non-finite right state", "right", ~np.isfinite(qr), True)]


def _pos(arr, what, side):
    # kernels.py:152-156
    return (f"nonpositive {what} on {side} side", side, ~(arr > FLOOR), False)


@dataclass(frozen=True)
class Solver:
    name: str
    num_eqn: int
    num_waves: int
    num_aux: int
    params: dict = field(default_factory=dict)

    def solve(self, ni, ql, qr, auxl, auxr):
        with np.errstate(all="ignore"):
            return _SOLVE[self.name](ni, ql, qr, auxl, auxr, self.params)

    def checks(self, ni, ql, qr, auxl, auxr):
        with np.errstate(all="ignore"):
            return _CHECK[self.name](ni, ql, qr, auxl, auxr, self.params)


def rp_advection(ni, ql, qr, auxl, auxr, p):
    """kernels.py:163-178 — one wave qr-ql at u (x) or v (y)."""
    sp = p["u"] if ni == 1 else p["v"]
    jump = qr - ql
    w = jump[np.newaxis]
    s = np.full((1,) + jump.shape[1:], sp, dtype=jump.dtype)
    return w, s, min(sp, 0.0) * jump, max(sp, 0.0) * jump


def _chk_advection(ni, ql, qr, auxl, auxr, p):
    return _finite_checks(ql, qr)


def acoustics_const_params(rho: float, bulk: float) -> dict:
    # kernels.py:112-118: c = sqrt(K/rho), Z = rho*c (Python floats)
    c = math.sqrt(bulk / rho)
    return {"c": c, "z": rho * c}


def rp_acoustics_const(ni, ql, qr, auxl, auxr, p):
    """kernels.py:181-213."""
    z, c = p["z"], p["c"]
    dp = qr[0] - ql[0]
    dn = qr[ni] - ql[ni]
    a1 = (-dp + z * dn) / (2.0 * z)
    a2 = (dp + z * dn) / (2.0 * z)
    w = np.zeros((2, 3) + dp.shape, dtype=dp.dtype)
    w[0, 0] = -z * a1
    w[0, ni] = a1
    w[1, 0] = z * a2
    w[1, ni] = a2
    s = np.empty((2,) + dp.shape, dtype=dp.dtype)
    s[0] = -c
    s[1] = c
    return w, s, -c * w[0], c * w[1]


def _chk_acoustics_const(ni, ql, qr, auxl, auxr, p):
    return _finite_checks(ql, qr)


def rp_acoustics_var(ni, ql, qr, auxl, auxr, p):
    """kernels.py:216-261 — aux = (rho, c) per cell."""
    zl = auxl[0] * auxl[1]
    zr = auxr[0] * auxr[1]
    cl, cr = auxl[1], auxr[1]
    dp = qr[0] - ql[0]
    dn = qr[ni] - ql[ni]
    den = zl + zr
    a1 = (-dp + zr * dn) / den
    a2 = (dp + zl * dn) / den
    w = np.zeros((2, 3) + dp.shape, dtype=dp.dtype)
    w[0, 0] = -zl * a1
    w[0, ni] = a1
    w[1, 0] = zr * a2
    w[1, ni] = a2
    s = np.empty((2,) + dp.shape, dtype=dp.dtype)
    s[0] = -cl
    s[1] = cr
    return w, s, -cl * w[0], cr * w[1]


def _chk_acoustics_var(ni, ql, qr, auxl, auxr, p):
    # kernels.py:235-237: for each side: density then sound speed
    return _finite_checks(ql, qr) + [
        _pos(auxl[0], "density", "left"), _pos(auxl[1], "sound speed", "left"),
        _pos(auxr[0], "density", "right"), _pos(auxr[1], "sound speed", "right")]


def _gas_primitives(q, ni, ti, gm1):
    rho = q[0]
    u = q[ni] / rho
    v = q[ti] / rho
    pr = gm1 * (q[3] - 0.5 * rho * (u * u + v * v))
    return rho, u, v, pr


def rp_euler_roe(ni, ql, qr, auxl, auxr, p):
    """kernels.py:264-340 — Roe, three waves, no entropy fix."""
    gm1 = p["gamma"] - 1.0
    ti = 3 - ni
    rl, ul, vl, pl = _gas_primitives(ql, ni, ti, gm1)
    rr, ur, vr, pr = _gas_primitives(qr, ni, ti, gm1)
    sl = np.sqrt(rl)
    sr = np.sqrt(rr)
    ws = sl + sr
    uh = (sl * ul + sr * ur) / ws
    vh = (sl * vl + sr * vr) / ws
    hh = (sl * (ql[3] + pl) / rl + sr * (qr[3] + pr) / rr) / ws
    kin = 0.5 * (uh * uh + vh * vh)
    c2 = gm1 * (hh - kin)
    ch = np.sqrt(c2)
    d0 = qr[0] - ql[0]
    dm = qr[ni] - ql[ni]
    dt_ = qr[ti] - ql[ti]
    de = qr[3] - ql[3]
    ash = dt_ - vh * d0
    amid = gm1 / c2 * ((hh - uh * uh) * d0 + uh * dm - (de - ash * vh))
    span = (dm - uh * d0) / ch
    apl = 0.5 * (span + d0 - amid)
    ami = d0 - amid - apl
    w = np.empty((3, 4) + d0.shape, dtype=d0.dtype)
    w[0, 0] = ami
    w[0, ni] = ami * (uh - ch)
    w[0, ti] = ami * vh
    w[0, 3] = ami * (hh - uh * ch)
    w[1, 0] = amid
    w[1, ni] = amid * uh
    w[1, ti] = amid * vh + ash
    w[1, 3] = amid * kin + ash * vh
    w[2, 0] = apl
    w[2, ni] = apl * (uh + ch)
    w[2, ti] = apl * vh
    w[2, 3] = apl * (hh + uh * ch)
    s = np.empty((3,) + d0.shape, dtype=d0.dtype)
    s[0] = uh - ch
    s[1] = uh
    s[2] = uh + ch
    neg = np.minimum(s, 0.0)
    pos = np.maximum(s, 0.0)
    amdq = neg[0] * w[0] + neg[1] * w[1] + neg[2] * w[2]
    apdq = pos[0] * w[0] + pos[1] * w[1] + pos[2] * w[2]
    return w, s, amdq, apdq


def _roe_c2(ni, ql, qr, gm1):
    ti = 3 - ni
    rl, ul, vl, pl = _gas_primitives(ql, ni, ti, gm1)
    rr, ur, vr, pr = _gas_primitives(qr, ni, ti, gm1)
    sl = np.sqrt(rl)
    sr = np.sqrt(rr)
    ws = sl + sr
    uh = (sl * ul + sr * ur) / ws
    vh = (sl * vl + sr * vr) / ws
    hh = (sl * (ql[3] + pl) / rl + sr * (qr[3] + pr) / rr) / ws
    return gm1 * (hh - 0.5 * (uh * uh + vh * vh)), (pl, pr)


def _chk_gas(ni, ql, qr, auxl, auxr, p):
    # kernels.py:274-301: finite, density L/R, pressure L/R, Roe c^2 > 0
    gm1 = p["gamma"] - 1.0
    c2, (pl, pr) = _roe_c2(ni, ql, qr, gm1)
    return _finite_checks(ql, qr) + [
        _pos(ql[0], "density", "left"), _pos(qr[0], "density", "right"),
        _pos(pl, "pressure", "left"), _pos(pr, "pressure", "right"),
        ("Roe-average sound speed is not real", None, ~(c2 > 0.0), False)]


def rp_euler_hlle(ni, ql, qr, auxl, auxr, p):
    """Euler HLLE (Einfeldt 1988): two waves bounding the Riemann fan.

    Builder-owned formula (no reference counterpart):
      per side: u_n, u_t, p (u_l, v_l, p_l) as reference kernels.py:282-285, c = sqrt(g p/rho)
      Roe averages u^, c^ as reference kernels.py:289-302
      s1 = min(u_l - c_l, u^ - c^),  s2 = max(u_r + c_r, u^ + c^)
      with df = f(q_r) - f(q_l), dq = q_r - q_l and the middle state
      q_m = (df - s2 q_r + s1 q_l) / (s1 - s2):
      W1 = q_m - q_l = (df - s2 dq) * (1/(s1 - s2))  at s1
      W2 = q_r - q_m = (s1 dq - df) * (1/(s1 - s2))  at s2
      (written on the jumps so a zero jump gives exactly zero waves)
    amdq/apdq = sum of min/max(s,0) W in wave order.
    """
    gam = p["gamma"]
    gm1 = gam - 1.0
    ti = 3 - ni
    rl, ul, vl, pl = _gas_primitives(ql, ni, ti, gm1)
    rr, ur, vr, pr = _gas_primitives(qr, ni, ti, gm1)
    cl = np.sqrt(gam * pl / rl)
    cr = np.sqrt(gam * pr / rr)
    sl = np.sqrt(rl)
    sr = np.sqrt(rr)
    iws = 1.0 / (sl + sr)
    uh = (sl * ul + sr * ur) * iws
    vh = (sl * vl + sr * vr) * iws
    hh = (sl * (ql[3] + pl) / rl + sr * (qr[3] + pr) / rr) * iws
    c2 = gm1 * (hh - 0.5 * (uh * uh + vh * vh))
    ch = np.sqrt(c2)
    s1 = np.minimum(ul - cl, uh - ch)
    s2 = np.maximum(ur + cr, uh + ch)
    # physical fluxes (normal/transverse slots as reference kernels.py:366-370)
    fl = np.empty_like(ql)
    fr = np.empty_like(qr)
    for f, q, u, pp in ((fl, ql, ul, pl), (fr, qr, ur, pr)):
        f[0] = q[ni]
        f[ni] = q[ni] * u + pp
        f[ti] = q[ti] * u
        f[3] = u * (q[3] + pp)
    inv = 1.0 / (s1 - s2)
    df = fr - fl
    dq = qr - ql
    w = np.empty((2, 4) + s1.shape, dtype=s1.dtype)
    w[0] = (df - s2 * dq) * inv     # = q_m - q_l
    w[1] = (s1 * dq - df) * inv     # = q_r - q_m
    s = np.stack([s1, s2])
    neg = np.minimum(s, 0.0)
    pos = np.maximum(s, 0.0)
    amdq = neg[0] * w[0] + neg[1] * w[1]
    apdq = pos[0] * w[0] + pos[1] * w[1]
    return w, s, amdq, apdq


def _chk_gas_hlle(ni, ql, qr, auxl, auxr, p):
    gm1 = p["gamma"] - 1.0
    ti = 3 - ni
    rl, ul, vl, pl = _gas_primitives(ql, ni, ti, gm1)
    rr, ur, vr, pr = _gas_primitives(qr, ni, ti, gm1)
    sl = np.sqrt(rl)
    sr = np.sqrt(rr)
    iws = 1.0 / (sl + sr)
    uh = (sl * ul + sr * ur) * iws
    vh = (sl * vl + sr * vr) * iws
    hh = (sl * (ql[3] + pl) / rl + sr * (qr[3] + pr) / rr) * iws
    c2 = gm1 * (hh - 0.5 * (uh * uh + vh * vh))
    return _finite_checks(ql, qr) + [
        _pos(ql[0], "density", "left"), _pos(qr[0], "density", "right"),
        _pos(pl, "pressure", "left"), _pos(pr, "pressure", "right"),
        ("Roe-average sound speed is not real", None, ~(c2 > 0.0), False)]


def rp_shallow_roe(ni, ql, qr, auxl, auxr, p):
    """Shallow water, Roe linearisation + Harten's entropy fix.

    Builder-owned formula (no reference counterpart),
    q = (h, h u, h v), gravity g:
      per side: r = 1/h, u_n = q[ni]*r, u_t = q[ti]*r, sq = sqrt(h), c = sqrt(g)*sq
      u^ = (sq_l u_l + sq_r u_r) * (1/(sq_l + sq_r))   (v^ likewise)
      c^ = sqrt(g * (0.5*(h_l + h_r)))
      a1 = ((u^ + c^) d0 - d1) * (0.5/c^),  a2 = d2 - v^ d0,
      a3 = (d1 - (u^ - c^) d0) * (0.5/c^)
      W1 = a1 (1, u^-c^, v^) @ u^-c^,  W2 = a2 (0,0,1) @ u^,
      W3 = a3 (1, u^+c^, v^) @ u^+c^
    Harten's entropy fix (Harten 1983; LeVeque 2002 §15.3.5) on the genuinely
    nonlinear families p = 1, 3, with the Harten–Hyman width taken from the
    one-sided characteristic speeds:  delta_p = max(0, lam_p(q_r) - lam_p(q_l)),
    lam_1 = u - c, lam_3 = u + c.  |s|_H = |s| if |s| >= delta else
    (s*s + delta*delta) / (2*delta).  Then
      amdq = sum_p 0.5*(s_p - |s_p|_H) W_p,  apdq = sum_p 0.5*(s_p + |s_p|_H) W_p
    (the shear family p = 2 uses |s|), so amdq + apdq = sum_p s_p W_p exactly
    as for the plain Roe split and the Roe property f(q_r)-f(q_l) still holds.
    The CFL maximum uses the unmodified Roe speeds.
    """
    grav = p["grav"]
    sqg = math.sqrt(grav)
    ti = 3 - ni
    hl, hr = ql[0], qr[0]
    rhl = 1.0 / hl
    rhr = 1.0 / hr
    ul = ql[ni] * rhl
    ur = qr[ni] * rhr
    vl = ql[ti] * rhl
    vr = qr[ti] * rhr
    sl = np.sqrt(hl)
    sr = np.sqrt(hr)
    iws = 1.0 / (sl + sr)
    uh = (sl * ul + sr * ur) * iws
    vh = (sl * vl + sr * vr) * iws
    ch = np.sqrt(grav * (0.5 * (hl + hr)))
    d0 = qr[0] - ql[0]
    d1 = qr[ni] - ql[ni]
    d2 = qr[ti] - ql[ti]
    i2c = 0.5 / ch
    s1 = uh - ch
    s3 = uh + ch
    a1 = (s3 * d0 - d1) * i2c
    a2 = d2 - vh * d0
    a3 = (d1 - s1 * d0) * i2c
    w = np.zeros((3, 3) + d0.shape, dtype=d0.dtype)
    w[0, 0] = a1
    w[0, ni] = a1 * s1
    w[0, ti] = a1 * vh
    w[1, ti] = a2
    w[2, 0] = a3
    w[2, ni] = a3 * s3
    w[2, ti] = a3 * vh
    s = np.stack([s1, uh, s3])
    # Harten entropy fix on families 1 and 3
    cl = sqg * sl
    cr = sqg * sr
    d1w = np.maximum(0.0, (ur - cr) - (ul - cl))
    d3w = np.maximum(0.0, (ur + cr) - (ul + cl))
    ab = np.abs(s)
    fixed = ab.copy()
    for k, dl in ((0, d1w), (2, d3w)):
        m = ab[k] < dl
        if m.any():
            fixed[k] = np.where(m, (s[k] * s[k] + dl * dl) / (2.0 * np.where(m, dl, 1.0)),
                                ab[k])
    am = 0.5 * (s - fixed)
    ap = 0.5 * (s + fixed)
    amdq = np.empty_like(ql)
    apdq = np.empty_like(ql)
    # W2 only has a transverse component; the zero slots are skipped
    amdq[0] = am[0] * w[0, 0] + am[2] * w[2, 0]
    amdq[ni] = am[0] * w[0, ni] + am[2] * w[2, ni]
    amdq[ti] = am[0] * w[0, ti] + am[1] * w[1, ti] + am[2] * w[2, ti]
    apdq[0] = ap[0] * w[0, 0] + ap[2] * w[2, 0]
    apdq[ni] = ap[0] * w[0, ni] + ap[2] * w[2, ni]
    apdq[ti] = ap[0] * w[0, ti] + ap[1] * w[1, ti] + ap[2] * w[2, ti]
    return w, s, amdq, apdq


def _chk_shallow(ni, ql, qr, auxl, auxr, p):
    return _finite_checks(ql, qr) + [
        _pos(ql[0], "depth", "left"), _pos(qr[0], "depth", "right")]


_SOLVE = {
    "advection": rp_advection,
    "acoustics-const": rp_acoustics_const,
    "acoustics-var": rp_acoustics_var,
    "euler": rp_euler_roe,
    "euler-hlle": rp_euler_hlle,
    "shallow-water-roe": rp_shallow_roe,
}
_CHECK = {
    "advection": _chk_advection,
    "acoustics-const": _chk_acoustics_const,
    "acoustics-var": _chk_acoustics_var,
    "euler": _chk_gas,
    "euler-hlle": _chk_gas_hlle,
    "shallow-water-roe": _chk_shallow,
}
_SHAPES = {  # (num_eqn, num_waves, num_aux)
    "advection": (1, 1, 0),
    "acoustics-const": (3, 2, 0),
    "acoustics-var": (3, 2, 2),
    "euler": (4, 3, 0),
    "euler-hlle": (4, 2, 0),
    "shallow-water-roe": (3, 3, 0),
}


def make_solver(name: str, **params) -> Solver:
    if name not in _SOLVE:
        raise ValueError(f"unknown kernel {name!r}")
    neq, mw, naux = _SHAPES[name]
    if name == "advection":
        prm = {"u": float(params["u"]), "v": float(params["v"])}
    elif name == "acoustics-const":
        prm = acoustics_const_params(float(params["rho"]), float(params["bulk"]))
    elif name in ("euler", "euler-hlle"):
        prm = {"gamma": float(params.get("gamma", 1.4))}
    elif name == "shallow-water-roe":
        prm = {"grav": float(params.get("grav", 9.81))}
    else:
        prm = {}
    return Solver(name, neq, mw, naux, prm)


# ---------------------------------------------------------------------------
# limiters and the second-order correction (LeVeque 1997 / 2002 §6.9, §21)


def phi(theta: np.ndarray, limiter: str) -> np.ndarray:
    if limiter == "minmod":
        return np.maximum(0.0, np.minimum(1.0, theta))
    if limiter == "superbee":
        return np.maximum(0.0, np.maximum(np.minimum(1.0, 2.0 * theta),
                                          np.minimum(2.0, theta)))
    if limiter == "mc":
        return np.maximum(0.0, np.minimum(np.minimum(0.5 * (1.0 + theta), 2.0),
                                          2.0 * theta))
    raise ValueError(f"unknown limiter {limiter!r}")


def _along(a, axis, lo, hi):
    idx = [slice(None)] * a.ndim
    idx[axis] = slice(lo, hi)
    return a[tuple(idx)]


def correction_flux(w, s, dtdn, limiter, axis):
    """F~ at the inner edges of an edge array solved on [-1, n+1].

    w (mw, neq, ...), s (mw, ...); `axis` is the sweep axis of w (2 or 3 for
    the edge index).  Wave p at edge k is compared with the same family at
    the upwind edge (k-1 if s_p > 0 else k+1):
        theta = (W_up . W) / (W . W)   (dot products summed m = 0..neq-1)
        W~ = phi(theta) W   (W~ = 0 when W . W == 0)
        F~ = 0.5 * sum_p ((|s_p| * (1 - dtdn |s_p|)) * phi_p) * W_p
    (the wave's scalar factors multiplied first: one product per component)
    Returns F~ for edges 1..nE-2 of the input (i.e. edges [0, n]).
    """
    mw, neq = w.shape[0], w.shape[1]
    n_e = w.shape[axis]
    own = _along(w, axis, 1, n_e - 1)
    lft = _along(w, axis, 0, n_e - 2)
    rgt = _along(w, axis, 2, n_e)
    so = _along(s, axis - 1, 1, n_e - 1)
    up = np.where((so > 0.0)[:, None], lft, rgt)
    dup = up[:, 0] * own[:, 0]
    dow = own[:, 0] * own[:, 0]
    for m in range(1, neq):
        dup = dup + up[:, m] * own[:, m]
        dow = dow + own[:, m] * own[:, m]
    nz = dow != 0.0
    theta = np.zeros_like(dow)
    np.divide(dup, dow, out=theta, where=nz)
    ph = phi(theta, limiter)
    a = np.abs(so)
    coef = a * (1.0 - dtdn * a)
    cph = coef * ph
    f = cph[0][None] * own[0]
    for p in range(1, mw):
        f = f + cph[p][None] * own[p]
    return 0.5 * f


# ---------------------------------------------------------------------------
# sweep + update over a band of rows


@dataclass
class Spec:
    nx: int
    ny: int
    dx: float
    dy: float
    g: int = 2


def _first_error(cands):
    """cands: (key tuple, direction, i, j, reason, side); min key wins."""
    best = min(cands, key=lambda c: c[0])
    raise OracleError(best[1], best[2], best[3], best[4], best[5])


def _collect(checks, dir_idx, width, i_of, j_of):
    """Error candidates ordered like reference CellWise/Serial sweeps.

    Chunks of MAX_BLOCK//width rows (sweep.py:117-120); inside a chunk the
    kernel's check order (stage), then first bad in C order over
    (component, i, j) (_first_bad, kernels.py:132-135).
    """
    rows_per = max(1, MAX_BLOCK // width)
    out = []
    for stage, (reason, side, mask, percomp) in enumerate(checks):
        if not mask.any():
            continue
        for idx in np.argwhere(mask):
            if percomp:
                comp, a, b = int(idx[0]), int(idx[1]), int(idx[2])
            else:
                comp, a, b = 0, int(idx[0]), int(idx[1])
            i, j = i_of(a), j_of(b)
            key = (dir_idx, j // rows_per, stage, comp, i, j)
            out.append((key, "xy"[dir_idx], i, j, reason, side))
    return out


class _BandResult:
    pass


def _solve_band(q, aux, spec: Spec, solver: Solver, ja: int, jb: int, order: int):
    """Pass 1 for rows [ja, jb): edge solves, band max |s|, error candidates."""
    g, nx, ny = spec.g, spec.nx, spec.ny
    ext = 1 if order == 2 else 0
    r = _BandResult()
    has_aux = aux is not None and aux.shape[0] > 0
    # x-edges i in [-ext, nx+ext], rows [ja, jb)
    i0, i1 = -ext, nx + ext
    ql = q[:, g + i0 - 1:g + i1, g + ja:g + jb]
    qr = q[:, g + i0:g + i1 + 1, g + ja:g + jb]
    al = aux[:, g + i0 - 1:g + i1, g + ja:g + jb] if has_aux else None
    ar = aux[:, g + i0:g + i1 + 1, g + ja:g + jb] if has_aux else None
    r.xw, r.xs, r.xm, r.xp = solver.solve(1, ql, qr, al, ar)
    # reference edge set i in [0, nx] only
    ref = slice(ext, ext + nx + 1)
    xs_ref = r.xs[:, ref]
    r.max_x = float(np.abs(xs_ref).max()) if xs_ref.size else 0.0
    cands = []
    chk = solver.checks(1, ql[:, ref], qr[:, ref],
                        al[:, ref] if has_aux else None, ar[:, ref] if has_aux else None)
    if any(c[2].any() for c in chk):
        cands += _collect(chk, 0, nx + 1, lambda a: a, lambda b: ja + b)
    # y-edges j in [ja-ext, jb+ext] (edge jb is shared with the next band)
    j0, j1 = ja - ext, jb + ext
    ql = q[:, g:g + nx, g + j0 - 1:g + j1]
    qr = q[:, g:g + nx, g + j0:g + j1 + 1]
    al = aux[:, g:g + nx, g + j0 - 1:g + j1] if has_aux else None
    ar = aux[:, g:g + nx, g + j0:g + j1 + 1] if has_aux else None
    r.yw, r.ys, r.ym, r.yp = solver.solve(2, ql, qr, al, ar)
    refy = slice(ext, ext + (jb - ja) + 1)
    ys_ref = r.ys[:, :, refy]
    r.max_y = float(np.abs(ys_ref).max()) if ys_ref.size else 0.0
    chk = solver.checks(2, ql[:, :, refy], qr[:, :, refy],
                        al[:, :, refy] if has_aux else None,
                        ar[:, :, refy] if has_aux else None)
    if any(c[2].any() for c in chk):
        cands += _collect(chk, 1, nx, lambda a: a, lambda b: ja + b)
    r.cands = cands
    r.ja, r.jb = ja, jb
    return r


def _update_band(q, spec: Spec, r: _BandResult, dt: float, order: int, limiter: str):
    """Pass 2: donor-cell update (sweep.py:271-277) + correction flux.

    Dimension by dimension: the reference's x term, then the x correction
    flux difference, then the y term and the y correction.  order=1 is the
    reference's update exactly (x term, then y term)."""
    g, nx = spec.g, spec.nx
    ja, jb = r.ja, r.jb
    nb = jb - ja
    ext = 1 if order == 2 else 0
    dtdx = dt / spec.dx
    dtdy = dt / spec.dy
    cells = q[:, g:g + nx, g + ja:g + jb]
    xm = r.xm[:, ext:ext + nx + 1]
    xp = r.xp[:, ext:ext + nx + 1]
    ym = r.ym[:, :, ext:ext + nb + 1]
    yp = r.yp[:, :, ext:ext + nb + 1]
    second = order == 2 and limiter != "none"
    cells -= dtdx * (xp[:, 0:nx] + xm[:, 1:nx + 1])
    if second:
        fx = correction_flux(r.xw, r.xs, dtdx, limiter, axis=2)
        cells -= dtdx * (fx[:, 1:nx + 1] - fx[:, 0:nx])
    cells -= dtdy * (yp[:, :, 0:nb] + ym[:, :, 1:nb + 1])
    if second:
        fy = correction_flux(r.yw, r.ys, dtdy, limiter, axis=3)
        cells -= dtdy * (fy[:, :, 1:nb + 1] - fy[:, :, 0:nb])


@dataclass
class Controller:
    """reference driver.py:17-31 (TimestepController)."""

    cfl: float = 0.9
    dt_max: float | None = None
    fixed_dt: float | None = None


def choose_dt(msx, msy, dx, dy, ctl: Controller, remaining=None) -> float:
    """reference driver.py:34-57, same operation order."""
    if ctl.fixed_dt is not None:
        dt = ctl.fixed_dt
    else:
        if msx < 0 or msy < 0:
            raise ValueError(f"wave speeds must be >= 0, got {msx}, {msy}")
        rate = msx / dx + msy / dy
        if rate == 0.0:
            raise ValueError("all wave speeds are zero; a stationary field needs fixed_dt")
        dt = ctl.cfl / rate
    if ctl.dt_max is not None:
        dt = min(dt, ctl.dt_max)
    if remaining is not None:
        dt = min(dt, remaining)
    return dt


@dataclass
class Report:
    dt: float
    cfl: float
    max_speed_x: float
    max_speed_y: float


_POOL: dict[int, ThreadPoolExecutor] = {}


def _pool(n):
    if n not in _POOL:
        _POOL[n] = ThreadPoolExecutor(max_workers=n)
    return _POOL[n]


def _bands(ny, nb):
    nb = max(1, min(nb, ny))
    step = -(-ny // nb)
    return [(a, min(a + step, ny)) for a in range(0, ny, step)]


def step(q, aux, spec: Spec, solver: Solver, ctl: Controller, *,
         bc_x=EXTRAPOLATE, bc_y=EXTRAPOLATE, order=1, limiter="none",
         remaining=None, threads=1) -> Report:
    """One ghost-fill / sweep / choose-dt / update cycle (driver.py:199-225).

    Mutates q.  order=1 reproduces the reference step bitwise; order=2 adds
    the limited correction flux.  threads>1 splits rows into bands executed
    by a thread pool (numpy releases the GIL), the same way the reference's
    StaticThreads backend does; results do not depend on the band split.
    """
    g = spec.g
    if order == 2 and g < 2:
        raise ValueError("second order needs num_ghost >= 2")
    fill_ghost(q, bc_x, bc_y, g)
    if aux is not None and aux.shape[0]:
        fill_ghost(aux, bc_x, bc_y, g)
    bands = _bands(spec.ny, threads)
    if threads > 1 and len(bands) > 1:
        res = list(_pool(threads).map(
            lambda b: _solve_band(q, aux, spec, solver, b[0], b[1], order), bands))
    else:
        res = [_solve_band(q, aux, spec, solver, a, b, order) for a, b in bands]
    cands = [c for r in res for c in r.cands]
    if cands:
        _first_error(cands)
    msx = max(r.max_x for r in res)
    msy = max(r.max_y for r in res)
    dt = choose_dt(msx, msy, spec.dx, spec.dy, ctl, remaining)
    if threads > 1 and len(res) > 1:
        list(_pool(threads).map(
            lambda r: _update_band(q, spec, r, dt, order, limiter), res))
    else:
        for r in res:
            _update_band(q, spec, r, dt, order, limiter)
    cfl = dt * (msx / spec.dx + msy / spec.dy)
    return Report(dt, cfl, msx, msy)


def run(q, aux, spec, solver, ctl, *, num_steps=None, t_final=None, **kw):
    """reference driver.py:228-250 loop (num_steps, or t_final with the
    1e-14*max(1, t_final) tolerance)."""
    reps = []
    if num_steps is not None:
        for _ in range(num_steps):
            reps.append(step(q, aux, spec, solver, ctl, **kw))
        return reps
    t = 0.0
    tol = 1e-14 * max(1.0, t_final)
    while t_final - t > tol:
        rep = step(q, aux, spec, solver, ctl, remaining=t_final - t, **kw)
        reps.append(rep)
        t += rep.dt
    return reps


def default_threads() -> int:
    return os.cpu_count() or 1
