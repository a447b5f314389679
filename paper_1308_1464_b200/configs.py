"""Seeded synthetic inputs for the five BASELINE.json configurations.

These stand in for the reference's benchmark cases (BASELINE.json
``configs[0..4]``; exact recipes in SURVEY.md §8(d)).  Arrays come back in
the reference's host layout: ``(ncomp, nx+2g, ny+2g)`` Fortran order with
zero ghosts (reference grid.py:76-95), interior cell (i, j) at
``[:, g+i, g+j]`` and cell centres x = x0 + (i + 1/2) dx.

Generation is plain numpy on the host (input preparation, not the hot
path); the 16384^2 scaling case can instead be generated on the device with
torch (``device=...``) because a 268 M-cell numpy Gaussian sum takes minutes
-- from the same numpy 1D factors, so the device field has the host's bits.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

G = 2  # ghost layers (reference num_ghost, grid.py:36)


@dataclass
class Case:
    name: str
    kernel: str
    kernel_params: dict
    nx: int
    ny: int
    dx: float
    dy: float
    limiter: str
    order: int
    cfl: float
    steps: int
    bc: str
    q: np.ndarray | None = None       # (neq, nx+4, ny+4) F-order
    aux: np.ndarray | None = None     # (naux, nx+4, ny+4) F-order or None
    dtype: str = "f64"
    meta: dict = field(default_factory=dict)

    @property
    def cells(self) -> int:
        return self.nx * self.ny


def _field(ncomp, nx, ny):
    return np.zeros((ncomp, nx + 2 * G, ny + 2 * G), order="F")


def _centres(nx, ny, dx, dy, x0=0.0, y0=0.0):
    x = x0 + (np.arange(nx) + 0.5) * dx
    y = y0 + (np.arange(ny) + 0.5) * dy
    return np.meshgrid(x, y, indexing="ij")


def c1_acoustics(n: int = 256, seed: int = 0, steps: int = 100) -> Case:
    """configs[0]: const acoustics, rho=1, K=4, Gaussian pressure + noise."""
    rng = np.random.default_rng(seed)
    dx = 1.0 / n
    xx, yy = _centres(n, n, dx, dx)
    q = _field(3, n, n)
    q[0, G:G + n, G:G + n] = (np.exp(-200.0 * ((xx - 0.5) ** 2 + (yy - 0.5) ** 2))
                              + rng.uniform(-1e-3, 1e-3, (n, n)))
    return Case("C1-acoustics-const", "acoustics-const", {"rho": 1.0, "bulk": 4.0},
                n, n, dx, dx, "mc", 2, 0.9, steps, "extrapolate", q)


def c2_shallow_water(n: int = 1024, seed: int = 0, steps: int = 200) -> Case:
    """configs[1]: radial dam break on [-1,1]^2, h = 2 (r<0.3) else 1, noise 1e-4."""
    rng = np.random.default_rng(seed)
    dx = 2.0 / n
    xx, yy = _centres(n, n, dx, dx, -1.0, -1.0)
    r = np.sqrt(xx * xx + yy * yy)
    q = _field(3, n, n)
    q[0, G:G + n, G:G + n] = np.where(r < 0.3, 2.0, 1.0) + rng.normal(0.0, 1e-4, (n, n))
    return Case("C2-shallow-water-roe", "shallow-water-roe", {"grav": 9.81},
                n, n, dx, dx, "mc", 2, 0.9, steps, "extrapolate", q)


def c3_euler_quadrants(n: int = 4096, seed: int = 0, steps: int = 50) -> Case:
    """configs[2]: four-quadrant Riemann data; quadrants drawn NE, NW, SW, SE."""
    rng = np.random.default_rng(seed)
    gamma = 1.4
    dx = 1.0 / n
    states = []
    for _ in range(4):
        rho = rng.uniform(0.1, 1.5)
        u = rng.uniform(-0.8, 0.8)
        v = rng.uniform(-0.8, 0.8)
        p = rng.uniform(0.1, 1.5)
        states.append((rho, rho * u, rho * v, p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v)))
    xx, yy = _centres(n, n, dx, dx)
    east, north = xx >= 0.5, yy >= 0.5
    masks = (east & north, ~east & north, ~east & ~north, east & ~north)
    q = _field(4, n, n)
    for k in range(4):
        inner = q[k, G:G + n, G:G + n]
        for m, st in zip(masks, states):
            inner[m] = st[k]
    return Case("C3-euler-hlle", "euler-hlle", {"gamma": gamma},
                n, n, dx, dx, "minmod", 2, 0.8, steps, "extrapolate", q,
                meta={"quadrant_states": states})


def _box5(a: np.ndarray) -> np.ndarray:
    """5x5 box filter with edge-replicate padding (separable, fixed order)."""
    p = np.pad(a, 2, mode="edge")
    r = p[0:-4] + p[1:-3] + p[2:-2] + p[3:-1] + p[4:]
    c = r[:, 0:-4] + r[:, 1:-3] + r[:, 2:-2] + r[:, 3:-1] + r[:, 4:]
    return c / 25.0


def c4_var_acoustics(n: int = 8192, seed: int = 0, steps: int = 50) -> Case:
    """configs[3]: lognormal (rho, K) smoothed 5x5; aux = (rho, c=sqrt(K/rho))."""
    rng = np.random.default_rng(seed)
    dx = 1.0 / n
    rho = _box5(rng.lognormal(0.0, 0.5, (n, n)))
    bulk = _box5(rng.lognormal(0.0, 0.5, (n, n)))
    x0, y0 = rng.uniform(0.25, 0.75, 2)
    sigma = 1.0 / 16.0
    xx, yy = _centres(n, n, dx, dx)
    q = _field(3, n, n)
    q[0, G:G + n, G:G + n] = np.exp(-((xx - x0) ** 2 + (yy - y0) ** 2) / (2.0 * sigma * sigma))
    aux = _field(2, n, n)
    aux[0, G:G + n, G:G + n] = rho
    aux[1, G:G + n, G:G + n] = np.sqrt(bulk / rho)
    return Case("C4-acoustics-var", "acoustics-var", {}, n, n, dx, dx, "mc", 2, 0.9,
                steps, "extrapolate", q, aux, meta={"pulse": (x0, y0)})


def c5_factors(nx: int, ny: int | None = None, seed: int = 0):
    """The 64-bump recipe's draws and its separable 1D factors (numpy).

    Returns (amp, ex, ey): ``amp`` (nb,), ``ex`` (nb, nx) = exp(-(x-x_k)^2/2w_k^2),
    ``ey`` (nb, ny) likewise in y.  Every generator of the C5 field (full grid
    on the host, a row band on the host, the full grid on the GPU) multiplies
    these same float64 factors in the same order, so all give the same bits.
    """
    ny = nx if ny is None else ny
    squares = max(1, ny // nx)
    rng = np.random.default_rng(seed)
    cen = rng.uniform(0.0, 1.0, (64 * squares, 2))
    amp = rng.uniform(0.05, 0.5, 64 * squares)
    wid = rng.uniform(0.01, 0.05, 64 * squares)
    cen[:, 1] += np.repeat(np.arange(squares), 64)
    dx = 1.0 / nx
    x = (np.arange(nx) + 0.5) * dx
    y = (np.arange(ny) + 0.5) * dx
    two_w2 = 2.0 * wid ** 2
    ex = np.exp(-((x[None, :] - cen[:, 0:1]) ** 2) / two_w2[:, None])
    ey = np.exp(-((y[None, :] - cen[:, 1:2]) ** 2) / two_w2[:, None])
    return amp, ex, ey


def c5_h_rows(nx: int, ny: int, j0: int, j1: int, seed: int = 0) -> np.ndarray:
    """Rows [j0, j1) of the C5 depth, h[i, j - j0] (numpy, bitwise equal to the
    same rows of the full field: h = 1 + sum_k amp_k (ex_k[i] ey_k[j]), k in
    draw order)."""
    amp, ex, ey = c5_factors(nx, ny, seed)
    h = np.ones((nx, j1 - j0))
    for k in range(amp.shape[0]):
        h += amp[k] * np.outer(ex[k], ey[k, j0:j1])
    return h


def c5_bumps(nx: int = 16384, ny: int | None = None, seed: int = 0, steps: int = 20,
             dtype: str = "f64", device=None, rows: tuple[int, int] | None = None) -> Case:
    """configs[4]: h = 1 + sum of 64 Gaussian bumps per unit square, hu = hv = 0.

    Weak scaling stacks unit squares along y (ny = nx*P, 64*P bumps, bump
    centres y offset by the square index).  Each bump is separable,
    exp(-(x-xk)^2/2w^2) * exp(-(y-yk)^2/2w^2) (stated choice: the product of
    the two 1D factors), summed bump by bump in draw order.  With ``device``
    set the sum runs in torch on that device from the same numpy factors (the
    same IEEE products and sums, so the same bits as the host) and the Case
    carries the device tensor in meta["h_dev"] ([j][i], fp64).  ``rows=(j0,
    j1)`` builds only that row band of the field as its own grid (the bounded
    CPU-baseline sample).
    """
    ny = nx if ny is None else ny
    squares = max(1, ny // nx)
    dx = 1.0 / nx
    j0, j1 = rows if rows is not None else (0, ny)
    name = "C5-shallow-water-scaling"
    case = Case(name, "shallow-water-roe", {"grav": 9.81},
                nx, j1 - j0, dx, dx, "mc", 2, 0.9, steps, "extrapolate", None,
                dtype=dtype, meta={"squares": squares, "rows": (j0, j1), "ny_full": ny})
    if device is None:
        q = _field(3, nx, j1 - j0)
        q[0, G:G + nx, G:G + (j1 - j0)] = c5_h_rows(nx, ny, j0, j1, seed)
        case.q = q
    else:
        import torch
        amp, ex, ey = c5_factors(nx, ny, seed)
        ext = torch.as_tensor(ex, device=device)
        eyt = torch.as_tensor(ey[:, j0:j1], device=device)
        h = torch.ones((j1 - j0, nx), dtype=torch.float64, device=device)  # [j][i]
        for k in range(amp.shape[0]):
            h += float(amp[k]) * torch.outer(eyt[k], ext[k])
        case.meta["h_dev"] = h
    return case


BUILDERS = {
    "c1": c1_acoustics,
    "c2": c2_shallow_water,
    "c3": c3_euler_quadrants,
    "c4": c4_var_acoustics,
    "c5": c5_bumps,
}


def bytes_per_cell(kernel: str, dtype: str = "f64") -> int:
    """Algorithmic bytes per cell-update: q read + aux read + q write."""
    neq = {"advection": 1, "acoustics-const": 3, "acoustics-var": 3, "euler": 4, "euler-hlle": 4,
           "shallow-water-roe": 3}[kernel]
    naux = 2 if kernel == "acoustics-var" else 0
    return (2 * neq + naux) * (8 if dtype == "f64" else 4)

