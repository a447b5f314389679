"""The candidate-filter CFL pre-pass (k_speeds_b) against the oracle.

The filter probes an edge exactly only when a cheap upper bound of its max
|s| reaches an exact lower bound of the step's maximum (the previous step's
argmax edge re-probed on the current state, running maxima); every other
edge provably cannot hold the maximum.  These cases aim at its corners:
a moving maximum (hint one step stale), all edges tied (every edge a
candidate), a single dominant edge, admissible cells outside the bound's
safe range (forced exact probes) and both precisions.  Bar: every dt and
max speed identical to the oracle, state bitwise.
"""

import numpy as np
import pytest

from helpers import device_run, oracle_run, same_bits

pytestmark = pytest.mark.gpu

NAME = "shallow-water-roe"


def _dam_break(nx, ny, seed=0):
    rng = np.random.default_rng(seed)
    dx, dy = 2.0 / nx, 2.0 / ny
    q = np.zeros((3, nx + 4, ny + 4), order="F")
    x = -1 + (np.arange(nx) + 0.5) * dx
    y = -1 + (np.arange(ny) + 0.5) * dy
    xx, yy = np.meshgrid(x, y, indexing="ij")
    q[0, 2:-2, 2:-2] = np.where(xx * xx + yy * yy < 0.09, 2.0, 1.0) + rng.normal(0, 1e-4, (nx, ny))
    return q, dx, dy


def _check(q, dx, dy, steps, *, order=2, limiter="mc", bc=("extrapolate", "extrapolate"),
           precision="f64", use_run=False):
    nx, ny = q.shape[1] - 4, q.shape[2] - 4
    oq, oreps = oracle_run(NAME, q, None, nx, ny, dx, dy, steps=steps, order=order,
                           limiter=limiter, bc_x=bc[0], bc_y=bc[1])
    dq, res, _ = device_run(NAME, q, None, nx, ny, dx, dy, steps=steps, order=order,
                            limiter=limiter, bc_x=bc[0], bc_y=bc[1], precision=precision,
                            use_run=use_run)
    assert res.error.code == 0 and res.steps_done == steps
    for k, (r, (dt, cfl, msx, msy)) in enumerate(zip(oreps, res.reports)):
        assert (r.dt, r.max_speed_x, r.max_speed_y) == (dt, msx, msy), f"step {k}"
    assert same_bits(oq, dq), f"max |diff| = {np.abs(oq - dq).max():.3e}"


def test_dam_break_moving_maximum():
    # C2's recipe at 200x170, 30 steps: the maximum sits on the expanding front
    q, dx, dy = _dam_break(200, 170, seed=3)
    _check(q, dx, dy, 30)
    _check(q, dx, dy, 30, use_run=True)


def test_all_edges_tied():
    # lake at rest: every edge has the same max |s| (all are candidates)
    nx, ny = 97, 61
    q = np.zeros((3, nx + 4, ny + 4), order="F")
    q[0] = 1.5
    _check(q, 1.0 / nx, 1.0 / ny, 3)


def test_single_dominant_edge_and_periodic():
    nx, ny = 131, 77
    q = np.zeros((3, nx + 4, ny + 4), order="F")
    q[0] = 1.0
    q[0, 2 + 100, 2 + 5] = 1.3
    q[1, 2 + 7, 2 + 70] = 0.4
    _check(q, 1.0 / nx, 1.0 / ny, 6, bc=("periodic", "periodic"))
    _check(q, 1.0 / nx, 1.0 / ny, 6, order=1, limiter="none")


def test_cells_outside_the_bound_range_are_probed():
    # admissible, but the seeds' safe range is left: h just above the 1e-300
    # floor, and momenta whose velocity bound exceeds 2^500 -> forced exact
    # probes; the step's maximum sits on those edges
    nx, ny = 64, 48
    rng = np.random.default_rng(5)
    q = np.zeros((3, nx + 4, ny + 4), order="F")
    q[0, 2:-2, 2:-2] = rng.uniform(1.0, 1.1, (nx, ny))
    q[0, 2 + 10, 2 + 10] = 1.2e-300
    q[1, 2 + 30, 2 + 20] = 1e155
    dx, dy = 1.0 / nx, 1.0 / ny
    oq, oreps = oracle_run(NAME, q, None, nx, ny, dx, dy, steps=1, order=1)
    dq, res, _ = device_run(NAME, q, None, nx, ny, dx, dy, steps=1, order=1)
    assert res.error.code == 0
    r = oreps[0]
    assert (r.dt, r.max_speed_x, r.max_speed_y) == tuple(res.reports[0][i] for i in (0, 2, 3))
    assert np.array_equal(oq, dq, equal_nan=True)


@pytest.mark.parametrize("seed", [11, 12])
def test_random_states_fp32(seed):
    q, dx, dy = _dam_break(150, 90, seed=seed)
    q[1, 2:-2, 2:-2] = np.random.default_rng(seed).uniform(-0.5, 0.5, (150, 90))
    q32 = np.asfortranarray(q, dtype=np.float32)
    nx, ny = 150, 90
    oq, oreps = oracle_run(NAME, q32, None, nx, ny, dx, dy, steps=8, order=2, limiter="mc")
    dq, res, _ = device_run(NAME, q32, None, nx, ny, dx, dy, steps=8, order=2, limiter="mc",
                            precision="f32")
    assert res.error.code == 0
    for r, (dt, cfl, msx, msy) in zip(oreps, res.reports):
        assert (r.dt, r.max_speed_x, r.max_speed_y) == (dt, msx, msy)
    assert same_bits(oq, dq)


def test_reupload_invalidates_tile_data():
    # tile maxima, hint edges and the lower bound describe the state the last
    # update wrote; a new upload on the same handle must not reuse them
    from helpers import device_grid
    from paper_1308_1464_b200 import _abi
    nx, ny = 120, 90
    q1, dx, dy = _dam_break(nx, ny, seed=1)
    q2 = np.zeros_like(q1)
    q2[0] = 1.0
    q2[0, 2 + 100, 2 + 80] = 3.0   # the only fast spot, far from q1's front
    g = device_grid(NAME, nx, ny, dx, dy, order=2, limiter="mc")
    try:
        ctl = _abi.make_ctl(0.9)
        g.upload(q1)
        for _ in range(4):
            g.step(ctl)
        g.poll()
        g.upload(q2)
        for _ in range(4):
            g.step(ctl)
        res = g.poll()
        out = g.download()
    finally:
        g.close()
    oq, oreps = oracle_run(NAME, q2, None, nx, ny, dx, dy, steps=4, order=2, limiter="mc")
    assert [(r.dt, r.max_speed_x, r.max_speed_y) for r in oreps] == \
        [(r[0], r[2], r[3]) for r in res.reports]
    assert same_bits(oq, out)


def test_many_tiles_two_fronts():
    # 900x700: 32x25 tiles, several candidate tiles far apart (two dams)
    nx, ny = 900, 700
    rng = np.random.default_rng(9)
    dx, dy = 1.0 / nx, 1.0 / ny
    q = np.zeros((3, nx + 4, ny + 4), order="F")
    x = (np.arange(nx) + 0.5) * dx
    y = (np.arange(ny) + 0.5) * dy
    xx, yy = np.meshgrid(x, y, indexing="ij")
    h = 1.0 + 0.6 * np.exp(-400 * ((xx - 0.2) ** 2 + (yy - 0.3) ** 2)) \
        + 0.59 * np.exp(-300 * ((xx - 0.8) ** 2 + (yy - 0.7) ** 2))
    q[0, 2:-2, 2:-2] = h + rng.normal(0, 1e-5, (nx, ny))
    _check(q, dx, dy, 12, bc=("periodic", "extrapolate"))


# ---- ideal gas (Euler Roe / HLLE): tile accumulators of u, v, c^2 and a
# "safe" flag (internal energy >= 2^-10 E, ranges); unsafe tiles probe all

def _gas(rho, u, v, p, gamma=1.4):
    return np.stack([rho, rho * u, rho * v, p / (gamma - 1) + 0.5 * rho * (u * u + v * v)])


def _check_gas(name, q, dx, dy, steps, *, order=2, limiter="minmod",
               bc=("extrapolate", "extrapolate"), precision="f64"):
    nx, ny = q.shape[1] - 4, q.shape[2] - 4
    if precision == "f32":
        q = np.asfortranarray(q, dtype=np.float32)
    oq, oreps = oracle_run(name, q, None, nx, ny, dx, dy, steps=steps, order=order,
                           limiter=limiter, bc_x=bc[0], bc_y=bc[1], cfl=0.8)
    dq, res, _ = device_run(name, q, None, nx, ny, dx, dy, steps=steps, order=order,
                            limiter=limiter, bc_x=bc[0], bc_y=bc[1], precision=precision, cfl=0.8)
    assert res.error.code == 0 and res.steps_done == steps
    for k, (r, (dt, cfl, msx, msy)) in enumerate(zip(oreps, res.reports)):
        assert (r.dt, r.max_speed_x, r.max_speed_y) == (dt, msx, msy), f"step {k}"
    assert same_bits(oq, dq), f"max |diff| = {np.abs(oq - dq).max():.3e}"


@pytest.mark.parametrize("name", ["euler", "euler-hlle"])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_gas_quadrants(name, precision):
    # the C3 recipe at 180x150: piecewise-constant quadrants, one fastest
    nx, ny = 180, 150
    rng = np.random.default_rng(33)
    q = np.zeros((4, nx + 4, ny + 4), order="F")
    x = (np.arange(nx) + 0.5) / nx
    y = (np.arange(ny) + 0.5) / ny
    xx, yy = np.meshgrid(x, y, indexing="ij")
    rho = np.empty((nx, ny)); u = np.empty_like(rho); v = np.empty_like(rho); p = np.empty_like(rho)
    for m in ((xx >= .5) & (yy >= .5), (xx < .5) & (yy >= .5), (xx < .5) & (yy < .5),
              (xx >= .5) & (yy < .5)):
        rho[m], u[m], v[m], p[m] = (rng.uniform(.1, 1.5), rng.uniform(-.8, .8),
                                    rng.uniform(-.8, .8), rng.uniform(.1, 1.5))
    q[:, 2:-2, 2:-2] = _gas(rho, u, v, p)
    _check_gas(name, q, 1 / nx, 1 / ny, 10, precision=precision)


@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("name", ["euler", "euler-hlle"])
def test_gas_high_mach_and_hot_spot(name, precision):
    # a Mach ~100 jet (internal energy below 2^-10 E: unsafe tiles, probed in
    # full), a hot spot far from it that holds the maximum, periodic x
    nx, ny = 160, 120
    rho = np.ones((nx, ny)); u = np.zeros((nx, ny)); v = np.zeros((nx, ny)); p = np.ones((nx, ny))
    u[20:40, 10:30] = 120.0
    p[120:126, 90:96] = 2.0e5
    q = np.zeros((4, nx + 4, ny + 4), order="F")
    q[:, 2:-2, 2:-2] = _gas(rho, u, v, p)
    _check_gas(name, q, 1 / nx, 1 / ny, 6, bc=("periodic", "extrapolate"), precision=precision)


def test_gas_contact_with_large_temperature_ratio():
    # density ratio 1e9 across a contact at rest: c^2 differs by 1e9 between
    # neighbours (the c^2 > 0 safety margin of the Roe average)
    nx, ny = 90, 64
    rho = np.where(np.arange(nx)[:, None] < 45, 1.0, 1e-9) * np.ones((nx, ny))
    q = np.zeros((4, nx + 4, ny + 4), order="F")
    q[:, 2:-2, 2:-2] = _gas(rho, np.zeros((nx, ny)), np.full((nx, ny), 0.1), np.ones((nx, ny)))
    _check_gas("euler-hlle", q, 1 / nx, 1 / ny, 5)


@pytest.mark.parametrize("name,steps", [("shallow-water-roe", 120), ("euler-hlle", 60),
                                        ("euler", 40)])
def test_long_runs_equal_the_exact_prepass(monkeypatch, name, steps):
    # many steps of an evolving flow at a size with hundreds of tiles: the
    # filtered pre-pass (default) against the probe-every-edge pre-pass,
    # device against device -- every report and the final state identical
    from helpers import device_run
    nx, ny = 640, 470
    if name == "shallow-water-roe":
        q, dx, dy = _dam_break(nx, ny, seed=8)
    else:
        rng = np.random.default_rng(8)
        dx, dy = 1 / nx, 1 / ny
        xx, yy = np.meshgrid((np.arange(nx) + .5) * dx, (np.arange(ny) + .5) * dy, indexing="ij")
        r2 = (xx - .4) ** 2 + (yy - .6) ** 2
        rho = np.where(r2 < .02, 2.0, 1.0) + rng.normal(0, 1e-4, (nx, ny))
        p = np.where(r2 < .02, 5.0, 1.0)
        q = np.zeros((4, nx + 4, ny + 4), order="F")
        q[:, 2:-2, 2:-2] = _gas(rho, 0.1 * np.ones_like(rho), np.zeros_like(rho), p)
    kw = dict(steps=steps, order=2, limiter="mc", bc_x="periodic", bc_y="extrapolate",
              use_run=True)
    monkeypatch.setenv("WS_SPEEDS", "exact")
    ref, rres, _ = device_run(name, q, None, nx, ny, dx, dy, **kw)
    monkeypatch.delenv("WS_SPEEDS")
    out, res, _ = device_run(name, q, None, nx, ny, dx, dy, **kw)
    assert res.error.code == 0 and res.steps_done == steps
    assert res.reports == rres.reports
    assert same_bits(ref, out)


def test_gas_error_in_a_far_tile_after_filtered_steps():
    # Roe without entropy fix in a strong 2D rarefaction (two streams moving
    # apart) turns inadmissible after a few steps, in tiles far from the hot
    # spot that holds the CFL maximum: the emptying tiles fall below the
    # "safe" internal-energy fraction, get probed, and the device stops at
    # the oracle's last good step with the same error text
    from helpers import device_grid
    from paper_1308_1464_b200 import SweepError, _abi
    from oracle import wavestep_oracle as O
    name, nx, ny = "euler", 200, 150
    rho = np.ones((nx, ny)); u = np.zeros((nx, ny)); v = np.zeros((nx, ny)); p = np.ones((nx, ny))
    u[20:60, 20:60] = np.where(np.arange(20, 60)[:, None] < 40, -2.0, 2.0)
    p[20:60, 20:60] = 0.2
    p[170:176, 120:126] = 300.0
    q = np.zeros((4, nx + 4, ny + 4), order="F")
    q[:, 2:-2, 2:-2] = _gas(rho, u, v, p)
    dx, dy = 1 / nx, 1 / ny
    oq = np.asfortranarray(q.copy())
    solver = O.make_solver(name, gamma=1.4)
    good, err = 0, None
    for _ in range(40):
        try:
            O.step(oq, None, O.Spec(nx, ny, dx, dy), solver, O.Controller(0.9),
                   bc_x="extrapolate", bc_y="extrapolate", order=2, limiter="mc")
            good += 1
        except O.OracleError as e:
            err = e
            break
    assert err is not None and good >= 2, "the rarefaction should fail after a few steps"
    g = device_grid(name, nx, ny, dx, dy, order=2, limiter="mc")
    try:
        g.upload(q, None)
        g.run(40, _abi.make_ctl(0.9))
        res = g.poll()
        assert res.steps_done == good and res.error.step == good
        with pytest.raises(SweepError) as de:
            g.raise_for(res.error)
        assert str(de.value) == str(err)
        out = g.download()
    finally:
        g.close()
    assert same_bits(out[:, 2:-2, 2:-2], oq[:, 2:-2, 2:-2])


@pytest.mark.parametrize("seed", range(6))
def test_random_configs_filtered_equals_exact(monkeypatch, seed):
    # randomised sizes (partial tiles, 1-tile-wide strips), boundary
    # conditions, limiters and precisions: the tile pre-pass against the
    # probe-every-edge pre-pass, device against device
    from helpers import device_run, random_state
    rng = np.random.default_rng(1000 + seed)
    name = ["shallow-water-roe", "euler-hlle", "euler"][seed % 3]
    nx, ny = int(rng.integers(20, 400)), int(rng.integers(20, 300))
    bc = [("extrapolate", "extrapolate"), ("periodic", "periodic"),
          ("periodic", "extrapolate")][int(rng.integers(0, 3))]
    limiter = ["minmod", "superbee", "mc"][int(rng.integers(0, 3))]
    precision = "f32" if rng.random() < 0.3 else "f64"
    q, _ = random_state(name, nx, ny, seed=seed)
    if precision == "f32":
        q = np.asfortranarray(q, dtype=np.float32)
    dx, dy = 1 / nx, 1 / ny
    kw = dict(steps=15, order=2, limiter=limiter, bc_x=bc[0], bc_y=bc[1], precision=precision)
    monkeypatch.setenv("WS_SPEEDS", "exact")
    ref, rres, _ = device_run(name, q, None, nx, ny, dx, dy, **kw)
    monkeypatch.delenv("WS_SPEEDS")
    out, res, _ = device_run(name, q, None, nx, ny, dx, dy, **kw)
    assert res.error.code == rres.error.code
    assert res.reports == rres.reports
    assert same_bits(ref, out)
