"""Anchors for the builder-owned oracle extension (CPU only).

No reference test pins SW-Roe+Harten, Euler-HLLE, the limiters or the
correction flux ("parity unpinned").  These checks anchor
them the way the reference anchors its own kernels (oracles.py:316-512):
fluctuation identity, Roe/conservation property, bitwise X/Y symmetry,
limiter known answers, periodic conservation, uniform fixed point, order-1
reduction, and Sod-tube accuracy against the exact Riemann solution.
"""

import json
import os
import hashlib

import numpy as np
import pytest

from helpers import PARAMS, oracle_run, random_state
from oracle import exact_riemann as X
from oracle import wavestep_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


def rel_err(v, ref):
    return float(np.max(np.abs(v - ref) / np.maximum(1.0, np.abs(ref))))


def gas(rng, n, g=1.4):
    rho = rng.uniform(0.1, 10.0, n)
    u, v = rng.uniform(-3, 3, n), rng.uniform(-3, 3, n)
    p = rng.uniform(0.1, 10.0, n)
    return np.stack([rho, rho * u, rho * v, p / (g - 1) + 0.5 * rho * (u * u + v * v)])


def sw(rng, n):
    h = rng.uniform(0.1, 5.0, n)
    return np.stack([h, h * rng.uniform(-2, 2, n), h * rng.uniform(-2, 2, n)])


def euler_flux(q, ni, g=1.4):
    ti = 3 - ni
    un = q[ni] / q[0]
    p = (g - 1) * (q[3] - 0.5 * (q[ni] ** 2 + q[ti] ** 2) / q[0])
    f = np.empty_like(q)
    f[0], f[ni], f[ti], f[3] = q[ni], q[ni] * un + p, q[ti] * un, un * (q[3] + p)
    return f


def sw_flux(q, ni, g=9.81):
    ti = 3 - ni
    un = q[ni] / q[0]
    f = np.empty_like(q)
    f[0], f[ni], f[ti] = q[ni], q[ni] * un + 0.5 * g * q[0] ** 2, q[ti] * un
    return f


@pytest.mark.parametrize("name", ["shallow-water-roe", "euler-hlle"])
def test_fluctuation_identity_and_roe_property(name):
    rng = np.random.default_rng(20240817)
    s = O.make_solver(name)
    for ni in (1, 2):
        ql = sw(rng, 5000) if name.startswith("shallow") else gas(rng, 5000)
        qr = sw(rng, 5000) if name.startswith("shallow") else gas(rng, 5000)
        w, sp, am, ap = s.solve(ni, ql, qr, None, None)
        wsum = sp[0][None] * w[0]
        for p in range(1, w.shape[0]):
            wsum = wsum + sp[p][None] * w[p]
        assert rel_err(am + ap, wsum) <= 1e-12
        flux = sw_flux if name.startswith("shallow") else euler_flux
        assert rel_err(am + ap, flux(qr, ni) - flux(ql, ni)) <= 1e-11


@pytest.mark.parametrize("name,swap", [("shallow-water-roe", [0, 2, 1]),
                                       ("euler-hlle", [0, 2, 1, 3])])
def test_xy_symmetry_bitwise(name, swap):
    rng = np.random.default_rng(10)
    ql = sw(rng, 200) if name.startswith("shallow") else gas(rng, 200)
    qr = sw(rng, 200) if name.startswith("shallow") else gas(rng, 200)
    s = O.make_solver(name)
    rx = s.solve(1, ql, qr, None, None)
    ry = s.solve(2, ql[swap], qr[swap], None, None)
    assert np.array_equal(rx[1], ry[1])
    assert np.array_equal(rx[2], ry[2][swap])
    assert np.array_equal(rx[3], ry[3][swap])


def test_harten_fix_only_acts_on_expansive_transonic_waves():
    s = O.make_solver("shallow-water-roe")
    # transonic rarefaction in family 1: u - c goes from -0.5 to +0.5
    g = 9.81
    hl, hr = 1.0, 0.6
    ul = np.sqrt(g * hl) - 0.5
    ur = np.sqrt(g * hr) + 0.5
    ql = np.array([[hl], [hl * ul], [0.0]])
    qr = np.array([[hr], [hr * ur], [0.0]])
    w, sp, am, ap = s.solve(1, ql, qr, None, None)
    plain = np.minimum(sp, 0)[:, None, :] * w
    assert not np.allclose(am, plain.sum(axis=0))      # fix active
    # a compressive (shock) jump keeps the plain Roe split
    ql2 = np.array([[1.0], [1.0], [0.0]])
    qr2 = np.array([[2.0], [0.0], [0.0]])
    w, sp, am, ap = s.solve(1, ql2, qr2, None, None)
    assert np.allclose(am, (np.minimum(sp, 0)[:, None, :] * w).sum(axis=0), rtol=0, atol=1e-15)


@pytest.mark.parametrize("lim,expect", [
    ("minmod", [0.0, 0.0, 0.5, 1.0, 1.0, 1.0]),
    ("superbee", [0.0, 0.0, 1.0, 1.0, 2.0, 2.0]),
    ("mc", [0.0, 0.0, 0.75, 1.0, 1.5, 2.0])])
def test_limiter_known_answers(lim, expect):
    theta = np.array([-1.0, 0.0, 0.5, 1.0, 2.0, 3.0])
    assert np.array_equal(O.phi(theta, lim), np.array(expect))


@pytest.mark.parametrize("name", ["shallow-water-roe", "euler-hlle", "acoustics-var", "euler"])
def test_periodic_second_order_conserves(name):
    nx, ny = 32, 24
    q, aux = random_state(name, nx, ny, 3)
    spec = O.Spec(nx, ny, 1 / nx, 1 / ny)
    s = O.make_solver(name, **({"gamma": 1.4} if "euler" in name else {}))
    q = np.asfortranarray(q)
    sums = q[:, 2:-2, 2:-2].sum(axis=(1, 2))
    for _ in range(10):
        O.step(q, aux, spec, s, O.Controller(0.9), bc_x="periodic", bc_y="periodic",
               order=2, limiter="mc")
        new = q[:, 2:-2, 2:-2].sum(axis=(1, 2))
        if name.startswith("acoustics"):
            # variable-coefficient acoustics is not in conservation form
            continue
        assert rel_err(new, sums) <= 1e-12
        sums = new


@pytest.mark.parametrize("name", ["shallow-water-roe", "euler-hlle"])
def test_uniform_state_is_a_fixed_point(name):
    nx, ny = 10, 6
    q = np.zeros((3 if name.startswith("shallow") else 4, nx + 4, ny + 4), order="F")
    if name.startswith("shallow"):
        q[:, 2:-2, 2:-2] = np.array([1.5, 0.3, -0.2])[:, None, None]
    else:
        q[:, 2:-2, 2:-2] = np.array([1.0, 0.1, 0.2, 2.5])[:, None, None]
    before = q.copy()
    r = O.step(q, None, O.Spec(nx, ny, 0.1, 0.1), O.make_solver(name), O.Controller(0.9),
               order=2, limiter="superbee")
    assert np.array_equal(q[:, 2:-2, 2:-2], before[:, 2:-2, 2:-2])
    assert r.cfl == pytest.approx(0.9, abs=1e-12)


def sod_l1(nx, order, limiter, solver="euler-hlle", t_final=0.15):
    from oracle.wavestep_oracle import run
    ny = 4
    q = np.zeros((4, nx + 4, ny + 4), order="F")
    x = (np.arange(nx) + 0.5) / nx
    left = x < 0.5
    for c, (a, b) in enumerate(zip((1.0, 0.0, 0.0, 2.5), (0.125, 0.0, 0.0, 0.25))):
        q[c, 2:-2, 2:-2] = np.where(left, a, b)[:, None]
    run(q, None, O.Spec(nx, ny, 1 / nx, 1 / nx), O.make_solver(solver), O.Controller(0.9),
        t_final=t_final, bc_x="extrapolate", bc_y="periodic", order=order, limiter=limiter)
    ex = X.sample((1.0, 0.0, 1.0), (0.125, 0.0, 0.1), 1.4, (x - 0.5) / t_final)
    return float(np.abs(q[0, 2:-2, 2] - ex[0]).sum() / nx)


def test_exact_riemann_star_state():
    # reference test_oracles.py:18-22 (Sod star state)
    p, u = X.star_state((1.0, 0.0, 1.0), (0.125, 0.0, 0.1), 1.4)
    assert p == pytest.approx(0.30313, abs=1e-4)
    assert u == pytest.approx(0.92745, abs=1e-4)


@pytest.mark.parametrize("order,limiter", [(1, "none"), (2, "minmod"), (2, "mc")])
def test_sod_accuracy_hlle(order, limiter):
    e400 = sod_l1(400, order, limiter)
    e800 = sod_l1(800, order, limiter)
    assert e400 <= 0.02
    assert e800 < e400


def test_limited_second_order_beats_first_order():
    assert sod_l1(400, 2, "mc") < sod_l1(400, 1, "none")


def test_oracle_golden_regression():
    """The extension's outputs are frozen in oracle_golden.json (regression)."""
    gold = json.load(open(os.path.join(HERE, "golden", "oracle_golden.json")))["steps"]
    for name, c in gold.items():
        if name == "c2-128":
            from paper_1308_1464_b200 import configs
            cs = configs.c2_shallow_water(128, steps=40)
            q, aux = cs.q, None
        else:
            q, aux = random_state(c["kernel"], c["nx"], c["ny"], c["seed"])
        oq, reps = oracle_run(c["kernel"], q, aux, c["nx"], c["ny"], c["dx"], c["dy"],
                              steps=c["steps"], order=c["order"], limiter=c["limiter"],
                              bc_x=c["bc_x"], bc_y=c["bc_y"], threads=3)
        assert [r.dt for r in reps] == c["dts"], name
        h = hashlib.sha256((np.asfortranarray(oq) + 0.0).tobytes(order="F")).hexdigest()
        assert h == c["q_sha256"], name


def test_oracle_matches_round1_fixture_dts():
    """The update's association changed after round 1 (x term + x correction,
    then y): every dt of the round-1 fixtures still agrees to 1e-12."""
    old = json.load(open(os.path.join(HERE, "golden", "oracle_golden_r1.json")))["steps"]
    new = json.load(open(os.path.join(HERE, "golden", "oracle_golden.json")))["steps"]
    assert old.keys() == new.keys()
    for name in old:
        a, b = np.array(old[name]["dts"]), np.array(new[name]["dts"])
        assert a.shape == b.shape
        assert np.abs(b / a - 1.0).max() <= 1e-12, name


@pytest.mark.parametrize("name,limiter", [("shallow-water-roe", "mc"),
                                          ("euler-hlle", "minmod"),
                                          ("euler", "superbee"),
                                          ("acoustics-var", "mc"),
                                          ("acoustics-const", "superbee")])
def test_oracle_second_order_equals_clawpack_order(name, limiter):
    """Independent anchor of the second-order update: the oracle
    against a Clawpack-grouped restatement (tests/clawpack_order.py), 10
    steps from the same state: relative state difference <= 1e-12 and every
    dt within 1e-12 (north_star's fp64 tolerance)."""
    import clawpack_order as CO
    nx, ny = 48, 37
    dx, dy = 1.0 / nx, 1.3 / ny
    q, aux = random_state(name, nx, ny, 11)
    solver = O.make_solver(name, **PARAMS[name])
    spec = O.Spec(nx, ny, dx, dy)
    oq = np.asfortranarray(q.copy())
    oa = np.asfortranarray(aux.copy()) if aux is not None else None
    cq = np.asfortranarray(q.copy())
    ca = np.asfortranarray(aux.copy()) if aux is not None else None
    for k in range(10):
        r = O.step(oq, oa, spec, solver, O.Controller(0.9), bc_x="periodic", bc_y="periodic",
                   order=2, limiter=limiter)
        dt, msx, msy = CO.step(cq, ca, nx, ny, dx, dy, solver, 0.9, "periodic", limiter)
        assert abs(r.dt / dt - 1.0) <= 1e-12, k
        assert abs(r.max_speed_x / msx - 1.0) <= 1e-12
    scale = np.abs(oq[:, 2:-2, 2:-2]).max(axis=(1, 2))
    rel = (np.abs(oq[:, 2:-2, 2:-2] - cq[:, 2:-2, 2:-2]).max(axis=(1, 2)) /
           np.where(scale > 0, scale, 1.0)).max()
    assert rel <= 1e-12, rel
    # and the two differ only by rounding, not identically (the check has teeth)
    assert not np.array_equal(oq, cq) or name.startswith("acoustics-const")
