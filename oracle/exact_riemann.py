"""Exact 1D Euler Riemann solution (test infrastructure only).

Classical pressure-function root solve (Toro, "Riemann Solvers and Numerical
Methods for Fluid Dynamics", ch. 4) — the same independent oracle role as
reference oracles.py:114-250 (exact_riemann_euler_1d), restated here so the
builder-owned HLLE / limiter extension can be anchored by the Sod L1 check
(reference sod_density_l1, oracles.py:495-512 pattern).
"""

from __future__ import annotations

import math

import numpy as np


def _branch(p, rho, pk, ck, g):
    if p > pk:   # shock
        a = 2.0 / ((g + 1.0) * rho)
        b = (g - 1.0) / (g + 1.0) * pk
        r = math.sqrt(a / (p + b))
        return (p - pk) * r, r * (1.0 - 0.5 * (p - pk) / (p + b))
    e = (g - 1.0) / (2.0 * g)  # rarefaction
    f = 2.0 * ck / (g - 1.0) * ((p / pk) ** e - 1.0)
    return f, (p / pk) ** (-(g + 1.0) / (2.0 * g)) / (rho * ck)


def star_state(left, right, g):
    """(p*, u*) for primitive left/right (rho, u, p)."""
    rl, ul, pl = left
    rr, ur, pr = right
    cl, cr = math.sqrt(g * pl / rl), math.sqrt(g * pr / rr)
    if 2.0 * (cl + cr) / (g - 1.0) <= ur - ul:
        raise ValueError("vacuum generated")
    p = max(1e-12, 0.5 * (pl + pr))
    for _ in range(100):
        fl, dl = _branch(p, rl, pl, cl, g)
        fr, dr = _branch(p, rr, pr, cr, g)
        step = (fl + fr + ur - ul) / (dl + dr)
        pn = max(1e-14, p - step)
        if abs(pn - p) <= 1e-14 * 0.5 * (pn + p):
            p = pn
            break
        p = pn
    fl, _ = _branch(p, rl, pl, cl, g)
    fr, _ = _branch(p, rr, pr, cr, g)
    return p, 0.5 * (ul + ur) + 0.5 * (fr - fl)


def sample(left, right, g, xi):
    """Primitive (rho, u, p) at similarity coordinates xi = x/t."""
    rl, ul, pl = left
    rr, ur, pr = right
    ps, us = star_state(left, right, g)
    cl, cr = math.sqrt(g * pl / rl), math.sqrt(g * pr / rr)
    out = np.empty((3, len(xi)))
    for k, s in enumerate(np.asarray(xi, dtype=float)):
        if s <= us:  # left of contact
            if ps > pl:
                sh = ul - cl * math.sqrt((g + 1) / (2 * g) * ps / pl + (g - 1) / (2 * g))
                if s <= sh:
                    out[:, k] = (rl, ul, pl)
                else:
                    rho = rl * ((ps / pl + (g - 1) / (g + 1)) / ((g - 1) / (g + 1) * ps / pl + 1))
                    out[:, k] = (rho, us, ps)
            else:
                cs = cl * (ps / pl) ** ((g - 1) / (2 * g))
                if s <= ul - cl:
                    out[:, k] = (rl, ul, pl)
                elif s >= us - cs:
                    out[:, k] = (rl * (ps / pl) ** (1 / g), us, ps)
                else:
                    c = 2 / (g + 1) * (cl + (g - 1) / 2 * (ul - s))
                    u = 2 / (g + 1) * (cl + (g - 1) / 2 * ul + s)
                    rho = rl * (c / cl) ** (2 / (g - 1))
                    out[:, k] = (rho, u, pl * (c / cl) ** (2 * g / (g - 1)))
        else:
            if ps > pr:
                sh = ur + cr * math.sqrt((g + 1) / (2 * g) * ps / pr + (g - 1) / (2 * g))
                if s >= sh:
                    out[:, k] = (rr, ur, pr)
                else:
                    rho = rr * ((ps / pr + (g - 1) / (g + 1)) / ((g - 1) / (g + 1) * ps / pr + 1))
                    out[:, k] = (rho, us, ps)
            else:
                cs = cr * (ps / pr) ** ((g - 1) / (2 * g))
                if s >= ur + cr:
                    out[:, k] = (rr, ur, pr)
                elif s <= us + cs:
                    out[:, k] = (rr * (ps / pr) ** (1 / g), us, ps)
                else:
                    c = 2 / (g + 1) * (cr - (g - 1) / 2 * (ur - s))
                    u = 2 / (g + 1) * (-cr + (g - 1) / 2 * ur + s)
                    rho = rr * (c / cr) ** (2 / (g - 1))
                    out[:, k] = (rho, u, pr * (c / cr) ** (2 * g / (g - 1)))
    return out
