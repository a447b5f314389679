"""Shared parity helpers: seeded inputs, an oracle run and a device run."""

from __future__ import annotations

import numpy as np

from oracle import wavestep_oracle as O

PARAMS = {
    "advection": {"u": 0.7, "v": -1.3},
    "acoustics-const": {"rho": 1.3, "bulk": 2.1},
    "acoustics-var": {},
    "euler": {"gamma": 1.4},
    "euler-hlle": {"gamma": 1.4},
    "shallow-water-roe": {"grav": 9.81},
}
SHAPES = {"advection": (1, 0), "acoustics-const": (3, 0), "acoustics-var": (3, 2), "euler": (4, 0),
          "euler-hlle": (4, 0), "shallow-water-roe": (3, 0)}


def random_state(name, nx, ny, seed=0, dtype=np.float64, smooth=True):
    """Admissible seeded state (+aux) in the reference layout (ncomp, nx+4, ny+4) F."""
    rng = np.random.default_rng(seed)
    neq, naux = SHAPES[name]
    q = np.zeros((neq, nx + 4, ny + 4), order="F")
    aux = np.zeros((naux, nx + 4, ny + 4), order="F") if naux else None
    xx, yy = np.meshgrid((np.arange(nx) + 0.5) / nx, (np.arange(ny) + 0.5) / ny, indexing="ij")
    bump = np.exp(-40.0 * ((xx - 0.4) ** 2 + (yy - 0.55) ** 2)) if smooth else 0.0
    I = (slice(None), slice(2, nx + 2), slice(2, ny + 2))
    if name == "advection":
        q[I] = rng.normal(0.0, 0.1, (1, nx, ny))
        q[0, 2:nx + 2, 2:ny + 2] += bump
    elif name in ("acoustics-const", "acoustics-var"):
        q[I] = rng.normal(0.0, 0.1, (3, nx, ny))
        q[0, 2:nx + 2, 2:ny + 2] += bump
        if naux:
            aux[0, 2:nx + 2, 2:ny + 2] = rng.uniform(0.5, 2.0, (nx, ny))
            aux[1, 2:nx + 2, 2:ny + 2] = rng.uniform(0.5, 2.0, (nx, ny))
    elif name in ("euler", "euler-hlle"):
        rho = rng.uniform(0.8, 1.2, (nx, ny)) + bump
        u = rng.uniform(-0.3, 0.3, (nx, ny))
        v = rng.uniform(-0.3, 0.3, (nx, ny))
        p = rng.uniform(0.8, 1.2, (nx, ny)) + bump
        q[I] = np.stack([rho, rho * u, rho * v, p / 0.4 + 0.5 * rho * (u * u + v * v)])
    else:
        h = rng.uniform(1.0, 1.2, (nx, ny)) + bump
        q[I] = np.stack([h, h * rng.uniform(-0.3, 0.3, (nx, ny)),
                         h * rng.uniform(-0.3, 0.3, (nx, ny))])
    if dtype != np.float64:
        q = np.asfortranarray(q, dtype=dtype)
        aux = np.asfortranarray(aux, dtype=dtype) if aux is not None else None
    return q, aux


def oracle_run(name, q, aux, nx, ny, dx, dy, *, steps, order=1, limiter="none",
               bc_x="extrapolate", bc_y="extrapolate", cfl=0.9, threads=1, **ctl):
    q = np.asfortranarray(q.copy())
    aux = np.asfortranarray(aux.copy()) if aux is not None else None
    solver = O.make_solver(name, **PARAMS[name])
    spec = O.Spec(nx, ny, dx, dy)
    c = O.Controller(cfl, ctl.get("dt_max"), ctl.get("fixed_dt"))
    reps = []
    for _ in range(steps):
        reps.append(O.step(q, aux, spec, solver, c, bc_x=bc_x, bc_y=bc_y, order=order,
                           limiter=limiter, threads=threads))
    return q, reps


def device_grid(name, nx, ny, dx, dy, *, order=1, limiter="none", bc_x="extrapolate",
                bc_y="extrapolate", precision="f64"):
    from paper_1308_1464_b200 import DeviceGrid, make_kernel
    return DeviceGrid(nx, ny, dx, dy, make_kernel(name, **PARAMS[name]), order=order,
                      limiter=limiter, bc_x=bc_x, bc_y=bc_y, precision=precision)


def device_run(name, q, aux, nx, ny, dx, dy, *, steps, order=1, limiter="none",
               bc_x="extrapolate", bc_y="extrapolate", cfl=0.9, precision="f64",
               use_run=False, **ctl):
    from paper_1308_1464_b200 import _abi
    g = device_grid(name, nx, ny, dx, dy, order=order, limiter=limiter, bc_x=bc_x,
                    bc_y=bc_y, precision=precision)
    try:
        g.upload(q, aux)
        c = _abi.make_ctl(cfl, ctl.get("dt_max"), ctl.get("fixed_dt"))
        if use_run:
            g.run(steps, c)
        else:
            for _ in range(steps):
                g.step(c)
        res = g.poll()
        out = g.download()
        return out, res, g.launches()
    finally:
        g.close()


def same_bits(a, b):
    """Value equality (the reference's own guard, bench.py:181: np.array_equal)."""
    return np.array_equal(a, b)


def case_oracle_run(case, steps, threads=None, dtype=np.float64):
    """Oracle run of a BASELINE recipe (paper_1308_1464_b200.configs.Case)."""
    import os
    q = np.asfortranarray(case.q, dtype=dtype).copy(order="F")
    aux = (np.asfortranarray(case.aux, dtype=dtype).copy(order="F")
           if case.aux is not None else None)
    solver = O.make_solver(case.kernel, **case.kernel_params)
    spec = O.Spec(case.nx, case.ny, case.dx, case.dy)
    c = O.Controller(case.cfl)
    reps = [O.step(q, aux, spec, solver, c, bc_x=case.bc, bc_y=case.bc, order=case.order,
                   limiter=case.limiter, threads=threads or os.cpu_count() or 1)
            for _ in range(steps)]
    return q, reps


def case_device_run(case, steps, precision="f64", use_run=True, download=True):
    """Device run of a BASELINE recipe through the C ABI (DeviceGrid)."""
    from paper_1308_1464_b200 import DeviceGrid, _abi, make_kernel
    g = DeviceGrid(case.nx, case.ny, case.dx, case.dy,
                   make_kernel(case.kernel, **case.kernel_params), order=case.order,
                   limiter=case.limiter, bc_x=case.bc, bc_y=case.bc, precision=precision)
    npdt = np.float64 if precision == "f64" else np.float32
    try:
        g.upload(np.asfortranarray(case.q, dtype=npdt),
                 np.asfortranarray(case.aux, dtype=npdt) if case.aux is not None else None)
        c = _abi.make_ctl(case.cfl)
        if use_run:
            g.run(steps, c)
        else:
            for _ in range(steps):
                g.step(c)
        res = g.poll()
        out = g.download() if download else None
        return out, res
    finally:
        g.close()


def assert_same_run(oq, oreps, dq, res, steps):
    """Bitwise state and identical dt / cfl / max speeds for every step."""
    assert res.error.code == 0, res.error
    assert res.steps_done == steps
    assert len(res.reports) == steps
    for k, (r, (dt, cfl, msx, msy)) in enumerate(zip(oreps, res.reports)):
        assert (r.dt, r.max_speed_x, r.max_speed_y, r.cfl) == (dt, msx, msy, cfl), f"step {k}"
    if not np.array_equal(oq, dq):
        d = np.abs(oq - dq)
        raise AssertionError(f"state differs: max |diff| {d.max():.3e} at "
                             f"{np.unravel_index(np.argmax(d), d.shape)}")
