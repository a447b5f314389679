"""An independent second-order step in Clawpack's grouping (test-only).

The production oracle (oracle/wavestep_oracle.py) fixes one association of
the second-order wave-propagation update so the CUDA kernels can match it
bit for bit.  This module restates the same published algorithm (LeVeque
1997; Clawpack step2 without transverse terms) with Clawpack's own grouping,
written independently of the oracle's update code:

* the limiter scales the wave first, W~_p = phi(theta_p) W_p, theta_p =
  (W_up . W_p) / (W_p . W_p) (Clawpack limiter: dotr / wnorm2);
* cqxx = sum_p |s_p| (1 - dtdx |s_p|) W~_p, F~ = cqxx / 2 (Clawpack flux2);
* one combined increment per direction, applied to q at once:
  q_new = q - dtdx (apdq_i + amdq_{i+1} + F~_{i+1} - F~_i)
            - dtdy (apdq_j + amdq_{j+1} + G~_{j+1} - G~_j).

Only the Riemann solvers (the physics plugins, pinned separately) and the
ghost fill are shared with the oracle.  The oracle and this step agree to
rounding, which tests/test_oracle_extension.py bounds: a reassociation of
the oracle made for speed cannot silently change the algorithm.
"""

from __future__ import annotations

import numpy as np

from oracle import wavestep_oracle as O


def _phi(th, limiter):
    if limiter == "minmod":
        return np.clip(th, 0.0, 1.0)
    if limiter == "superbee":
        return np.maximum.reduce([np.zeros_like(th), np.minimum(2.0 * th, 1.0),
                                  np.minimum(th, 2.0)])
    if limiter == "mc":
        return np.maximum(0.0, np.minimum.reduce([(1.0 + th) / 2.0, np.full_like(th, 2.0),
                                                  2.0 * th]))
    raise ValueError(limiter)


def _limited_flux(w, s, dtdn, limiter):
    """w (mw, neq, nE, ...) along axis 2, s (mw, nE, ...): F~ at edges 1..nE-2."""
    mw = w.shape[0]
    f = np.zeros((w.shape[1], w.shape[2] - 2) + w.shape[3:])
    for p in range(mw):
        wp = w[p]                         # (neq, nE, ...)
        sp = s[p]                         # (nE, ...)
        wnorm2 = np.einsum("m...,m...->...", wp[:, 1:-1], wp[:, 1:-1])
        up = np.where(sp[1:-1] > 0.0, 1, 0)
        dotr = np.where(up == 1,
                        np.einsum("m...,m...->...", wp[:, :-2], wp[:, 1:-1]),
                        np.einsum("m...,m...->...", wp[:, 2:], wp[:, 1:-1]))
        th = np.divide(dotr, wnorm2, out=np.zeros_like(dotr), where=wnorm2 != 0.0)
        wl = _phi(th, limiter)[None] * wp[:, 1:-1]          # W~ = phi W
        a = np.abs(sp[1:-1])
        f += (a * (1.0 - dtdn * a))[None] * wl
    return f / 2.0


def step(q, aux, nx, ny, dx, dy, solver, cfl, bc, limiter):
    """One second-order step; mutates q (ghost frame and interior)."""
    g = 2
    O.fill_ghost(q, bc, bc)
    if aux is not None:
        O.fill_ghost(aux, bc, bc)
    # x-edges i in [-1, nx+1] for every interior row, y-edges likewise
    xl, xr = q[:, g - 2:g + nx + 1, g:g + ny], q[:, g - 1:g + nx + 2, g:g + ny]
    yl, yr = q[:, g:g + nx, g - 2:g + ny + 1], q[:, g:g + nx, g - 1:g + ny + 2]
    ax = (aux[:, g - 2:g + nx + 1, g:g + ny], aux[:, g - 1:g + nx + 2, g:g + ny]) \
        if aux is not None else (None, None)
    ay = (aux[:, g:g + nx, g - 2:g + ny + 1], aux[:, g:g + nx, g - 1:g + ny + 2]) \
        if aux is not None else (None, None)
    xw, xs, xm, xp = solver.solve(1, xl, xr, *ax)
    yw, ys, ym, yp = solver.solve(2, yl, yr, *ay)
    msx = float(np.abs(xs[:, 1:nx + 2]).max())
    msy = float(np.abs(ys[:, :, 1:ny + 2]).max())
    dt = cfl / (msx / dx + msy / dy)
    dtdx, dtdy = dt / dx, dt / dy
    fx = _limited_flux(xw, xs, dtdx, limiter)                 # edges i = 0..nx
    fy = np.moveaxis(_limited_flux(np.moveaxis(yw, 3, 2), np.moveaxis(ys, 2, 1), dtdy,
                                   limiter), 1, 2)            # edges j = 0..ny
    incx = xp[:, 1:nx + 1] + xm[:, 2:nx + 2] + fx[:, 1:] - fx[:, :-1]
    incy = yp[:, :, 1:ny + 1] + ym[:, :, 2:ny + 2] + fy[:, :, 1:] - fy[:, :, :-1]
    q[:, g:g + nx, g:g + ny] -= dtdx * incx + dtdy * incy
    return dt, msx, msy
