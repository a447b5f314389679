"""GPU parity: the CUDA step against the numpy oracle, through the C ABI.

Bar (north_star): fp64 results identical to the oracle — bitwise, checked
with np.array_equal like the reference's own guard (bench.py:181) — and
every dt identical.  Sizes are deliberately not multiples of the 32x16
CUDA tile so partial tiles and the boundary index mapping are exercised.
"""

import numpy as np
import pytest

from helpers import PARAMS, device_run, oracle_run, random_state, same_bits
from oracle import wavestep_oracle as O

pytestmark = pytest.mark.gpu

SOLVERS = ["advection", "acoustics-const", "acoustics-var", "euler", "euler-hlle",
           "shallow-water-roe"]
BCS = [("extrapolate", "extrapolate"), ("periodic", "periodic"), ("periodic", "extrapolate")]


def _compare(name, nx, ny, steps, order, limiter, bc, seed=0, use_run=False, cfl=0.9):
    dx, dy = 1.0 / nx, 1.3 / ny
    q, aux = random_state(name, nx, ny, seed)
    oq, oreps = oracle_run(name, q, aux, nx, ny, dx, dy, steps=steps, order=order,
                           limiter=limiter, bc_x=bc[0], bc_y=bc[1], cfl=cfl)
    dq, res, _ = device_run(name, q, aux, nx, ny, dx, dy, steps=steps, order=order,
                            limiter=limiter, bc_x=bc[0], bc_y=bc[1], cfl=cfl, use_run=use_run)
    assert res.error.code == 0
    assert res.steps_done == steps
    for k, (r, (dt, cfl_r, msx, msy)) in enumerate(zip(oreps, res.reports)):
        assert (r.dt, r.max_speed_x, r.max_speed_y) == (dt, msx, msy), f"step {k}"
        assert r.cfl == cfl_r
    assert same_bits(oq, dq), f"max |diff| = {np.abs(oq - dq).max():.3e}"


@pytest.mark.parametrize("bc", BCS)
@pytest.mark.parametrize("name", SOLVERS)
def test_first_order_bitwise(name, bc):
    _compare(name, 37, 29, 4, 1, "none", bc)


@pytest.mark.parametrize("limiter", ["minmod", "superbee", "mc"])
@pytest.mark.parametrize("name", SOLVERS)
def test_second_order_bitwise(name, limiter):
    _compare(name, 45, 35, 4, 2, limiter, ("extrapolate", "extrapolate"), seed=1)


@pytest.mark.parametrize("name", ["shallow-water-roe", "euler-hlle", "acoustics-var"])
def test_second_order_periodic_bitwise(name):
    _compare(name, 40, 33, 4, 2, "mc", ("periodic", "periodic"), seed=2)


@pytest.mark.parametrize("name,bc", [("shallow-water-roe", "periodic"),
                                     ("euler-hlle", "extrapolate"), ("euler", "periodic")])
def test_many_tiles_bitwise(name, bc):
    # several tile rows/columns, partial edge tiles, periodic wrap borders: the
    # fused next-step CFL epilogue (shared-border counters) must give every dt
    _compare(name, 131, 75, 6, 2, "mc", (bc, bc), seed=9)
    _compare(name, 131, 75, 6, 2, "mc", (bc, bc), seed=9, use_run=True)


@pytest.mark.parametrize("name", ["shallow-water-roe", "acoustics-const"])
def test_graph_run_equals_steps(name):
    _compare(name, 64, 48, 9, 2, "mc", ("extrapolate", "extrapolate"), seed=3, use_run=True)


def test_tiny_grids():
    for nx, ny in ((1, 1), (2, 3), (5, 1), (33, 17)):
        _compare("shallow-water-roe", nx, ny, 3, 2, "mc", ("extrapolate", "extrapolate"), seed=4)
        _compare("acoustics-const", nx, ny, 3, 1, "none", ("extrapolate", "extrapolate"), seed=4)
    _compare("euler-hlle", 2, 2, 3, 2, "minmod", ("periodic", "periodic"), seed=5)


@pytest.mark.parametrize("name", SOLVERS)
def test_fp32_bitwise_vs_fp32_oracle(name):
    nx, ny = 50, 42
    dx = dy = 1.0 / 50
    q, aux = random_state(name, nx, ny, 6, dtype=np.float32)
    oq, oreps = oracle_run(name, q, aux, nx, ny, dx, dy, steps=5, order=2, limiter="mc")
    assert oq.dtype == np.float32
    dq, res, _ = device_run(name, q, aux, nx, ny, dx, dy, steps=5, order=2, limiter="mc",
                            precision="f32")
    assert [r.dt for r in oreps] == [r[0] for r in res.reports]
    assert same_bits(oq, dq)


def test_fp32_close_to_fp64():
    name, nx, ny = "shallow-water-roe", 64, 64
    dx = dy = 1.0 / 64
    q, _ = random_state(name, nx, ny, 7)
    q64, _ = oracle_run(name, q, None, nx, ny, dx, dy, steps=20, order=2, limiter="mc")
    q32, _, _ = device_run(name, np.asfortranarray(q, dtype=np.float32), None, nx, ny, dx, dy,
                           steps=20, order=2, limiter="mc", precision="f32")
    h64, h32 = q64[0, 2:-2, 2:-2], q32[0, 2:-2, 2:-2].astype(np.float64)
    rel = np.abs(h32 - h64).max() / np.abs(h64).max()
    assert rel <= 1e-5, rel   # stated fp32 bound


@pytest.mark.parametrize("name", SOLVERS)
def test_inadmissible_cell_reports_reference_location(name):
    from paper_1308_1464_b200 import SweepError
    from helpers import device_grid
    from paper_1308_1464_b200 import _abi
    nx, ny = 12, 9
    q, aux = random_state(name, nx, ny, 8)
    if name.startswith("acoustics"):
        q[1, 2 + 5, 2 + 3] = np.nan
    elif name == "advection":
        q[0, 2 + 5, 2 + 3] = np.inf
    else:
        q[0, 2 + 5, 2 + 3] = -1.0
    with pytest.raises(O.OracleError) as oe:
        oracle_run(name, q, aux, nx, ny, 1.0 / nx, 1.0 / ny, steps=1)
    g = device_grid(name, nx, ny, 1.0 / nx, 1.0 / ny)
    g.upload(q, aux)
    g.step(_abi.make_ctl(0.9))
    res = g.poll()
    with pytest.raises(SweepError) as de:
        g.raise_for(res.error)
    assert str(de.value) == str(oe.value)
    # state untouched: the download is the uploaded state with its ghosts filled
    out = g.download()
    assert np.array_equal(out[:, 2:-2, 2:-2], q[:, 2:-2, 2:-2], equal_nan=True)
    g.close()


def test_error_in_later_step_keeps_last_good_state():
    """A run that turns inadmissible mid-way stops at the last good state."""
    from helpers import device_grid
    from paper_1308_1464_b200 import _abi
    name, nx, ny = "euler", 24, 16
    rng = np.random.default_rng(11)
    q = np.zeros((4, nx + 4, ny + 4), order="F")
    rho = rng.uniform(0.1, 10, (nx, ny))
    u = rng.uniform(-3, 3, (nx, ny))
    v = rng.uniform(-3, 3, (nx, ny))
    p = rng.uniform(0.1, 10, (nx, ny))
    q[:, 2:-2, 2:-2] = np.stack([rho, rho * u, rho * v, p / 0.4 + 0.5 * rho * (u * u + v * v)])
    oq = np.asfortranarray(q.copy())
    solver = O.make_solver(name, gamma=1.4)
    good = 0
    err = None
    for _ in range(6):
        try:
            O.step(oq, None, O.Spec(nx, ny, 1 / nx, 1 / ny), solver, O.Controller(0.9),
                   bc_x="periodic", bc_y="periodic")
            good += 1
        except O.OracleError as e:
            err = e
            break
    assert err is not None, "input should turn inadmissible within 6 steps"
    g = device_grid(name, nx, ny, 1 / nx, 1 / ny, bc_x="periodic", bc_y="periodic")
    g.upload(q, None)
    g.run(6, _abi.make_ctl(0.9))
    res = g.poll()
    assert res.steps_done == good
    assert res.error.step == good
    out = g.download()
    assert same_bits(out[:, 2:-2, 2:-2], oq[:, 2:-2, 2:-2])
    g.close()


def test_fixed_dt_bypasses_the_cfl_formula():
    from helpers import device_grid
    from paper_1308_1464_b200 import _abi
    nx = ny = 8
    qa = np.zeros((3, nx + 4, ny + 4), order="F")
    aux = np.ones((2, nx + 4, ny + 4), order="F")
    g = device_grid("acoustics-var", nx, ny, 0.1, 0.1)
    g.upload(qa, aux)
    g.step(_abi.make_ctl(0.9, fixed_dt=1e-3))
    res = g.poll()
    assert res.error.code == 0 and res.reports[-1][0] == 1e-3
    # reference cfl = dt * (max_sx/dx + max_sy/dy) with max speeds c = 1
    assert res.reports[-1][1] == 1e-3 * (1.0 / 0.1 + 1.0 / 0.1)
    g.close()


def test_dt_max_remaining_and_fixed_dt_match_oracle():
    name, nx, ny = "shallow-water-roe", 30, 20
    q, _ = random_state(name, nx, ny, 12)
    for kw in ({"dt_max": 1e-4}, {"fixed_dt": 2.5e-4}):
        oq, oreps = oracle_run(name, q, None, nx, ny, 1 / nx, 1 / ny, steps=3, order=2,
                               limiter="superbee", **kw)
        dq, res, _ = device_run(name, q, None, nx, ny, 1 / nx, 1 / ny, steps=3, order=2,
                                limiter="superbee", **kw)
        assert [r.dt for r in oreps] == [r[0] for r in res.reports]
        assert same_bits(oq, dq)


# ---------------------------------------------------------------------------
# the device against the REFERENCE's own outputs (tests/golden, generated by
# running wavesweep itself) — no oracle in between

import hashlib
import json
import os

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                   "reference_golden.json")))


def _hash(q):
    return hashlib.sha256((np.asfortranarray(q, dtype=np.float64) + 0.0).tobytes(order="F")).hexdigest()


@pytest.mark.parametrize("name", sorted(GOLD["steps"]))
def test_device_matches_reference_golden(name):
    from paper_1308_1464_b200 import DeviceGrid, _abi, make_kernel
    c = GOLD["steps"][name]
    if name == "c1-full":
        from paper_1308_1464_b200 import configs
        q, aux = configs.c1_acoustics().q, None
    else:
        q, aux = random_state(c["kernel"], c["nx"], c["ny"], c["seed"])
    g = DeviceGrid(c["nx"], c["ny"], c["dx"], c["dy"], make_kernel(c["kernel"], **c["params"]),
                   order=1, bc_x=c["bc_x"], bc_y=c["bc_y"])
    g.upload(q, aux)
    g.run(c["steps"], _abi.make_ctl(0.9))
    res = g.poll()
    out = g.download()
    g.close()
    assert [r[0] for r in res.reports] == c["dts"]
    assert [r[2] for r in res.reports] == c["msx"]
    assert [r[3] for r in res.reports] == c["msy"]
    assert _hash(out) == c["q_sha256"]


@pytest.mark.parametrize("key", sorted(GOLD["kernels"]))
def test_device_kernel_solve_matches_reference(key):
    from paper_1308_1464_b200 import Direction, make_kernel
    c = GOLD["kernels"][key]
    name, d = key.rsplit("-", 1)
    k = make_kernel(name, **c["params"])
    r = k.solve(Direction.X if d == "x" else Direction.Y, np.array(c["ql"]), np.array(c["qr"]),
                np.array(c["auxl"]) if "auxl" in c else None,
                np.array(c["auxr"]) if "auxr" in c else None)
    assert np.array_equal(r.amdq, np.array(c["amdq"]))
    assert np.array_equal(r.apdq, np.array(c["apdq"]))
    assert np.array_equal(r.speeds, np.array(c["speeds"]))
    assert np.array_equal(r.waves, np.array(c["waves"]))


@pytest.mark.parametrize("key", sorted(GOLD["errors"]))
def test_device_error_text_matches_reference(key):
    from paper_1308_1464_b200 import (BoundaryCondition, GridSpec, SimulationConfig, StateField,
                                      AuxField, SweepError, TimestepController, step)
    from paper_1308_1464_b200.kernels import DESCRIPTORS
    c = GOLD["errors"][key]
    q, aux = random_state(c["kernel"], c["nx"], c["ny"], c["seed"])
    q[c["comp"], 2 + 5, 2 + 3] = float(eval(c["value"], {"nan": np.nan, "inf": np.inf}))
    d = DESCRIPTORS[c["kernel"]]
    spec = GridSpec(nx=c["nx"], ny=c["ny"], dx=1 / c["nx"], dy=1 / c["ny"], num_eqn=d.num_eqn,
                    num_aux=d.num_aux)
    st, ax = StateField(spec), AuxField(spec)
    st.data[...] = q
    if aux is not None:
        ax.data[...] = aux
    cfg = SimulationConfig(spec=spec, kernel=c["kernel"], ic="x", num_steps=1,
                           bc_x=BoundaryCondition.EXTRAPOLATE,
                           bc_y=BoundaryCondition.EXTRAPOLATE, kernel_params=c["params"])
    with pytest.raises(SweepError) as e:
        step(st, ax, cfg, TimestepController(0.9))
    assert str(e.value) == c["message"]


@pytest.mark.parametrize("name", ["euler-hlle", "shallow-water-roe", "acoustics-var"])
def test_tile_kernel_alternative_bitwise(monkeypatch, name):
    # the shared-memory tile kernel (WS_KERNEL=tile; the default is the
    # warp-line kernel for every solver) stays bitwise equal to the oracle
    monkeypatch.setenv("WS_KERNEL", "tile")
    _compare(name, 67, 53, 4, 2, "mc", ("periodic", "extrapolate"), seed=14)
    _compare(name, 67, 53, 3, 2, "minmod", ("extrapolate", "periodic"), seed=15, use_run=True)


def test_async_download_and_cross_stream_order():
    # uploads on one stream, steps + enqueue-only downloads on another: the
    # handle keeps issue order, so every downloaded state is the oracle's
    import torch
    from paper_1308_1464_b200 import _abi
    from helpers import device_grid
    name, nx, ny = "shallow-water-roe", 61, 43
    q, _ = random_state(name, nx, ny, 17)
    oq, _ = oracle_run(name, q, None, nx, ny, 1 / nx, 1.3 / ny, steps=2, order=2, limiter="mc")
    g = device_grid(name, nx, ny, 1 / nx, 1.3 / ny, order=2, limiter="mc")
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    outs = [torch.empty(3 * (nx + 4) * (ny + 4), dtype=torch.float64).pin_memory().numpy()
            .reshape((3, nx + 4, ny + 4), order="F") for _ in range(4)]
    try:
        ctl = _abi.make_ctl(0.9)
        for k in range(4):
            g.upload(q, None, stream=a.cuda_stream)
            g.step(ctl, stream=b.cuda_stream)
            g.step(ctl, stream=b.cuda_stream)
            g.download(outs[k], stream=b.cuda_stream, wait=False)
        torch.cuda.synchronize()
        assert g.poll().error.code == 0
        for o in outs:
            assert same_bits(oq, o)
        with pytest.raises(ValueError, match="async download needs"):
            g.download(np.zeros((3, nx + 4, ny + 4)), wait=False)
    finally:
        g.close()


@pytest.mark.parametrize("kernel_env,name", [("line", "shallow-water-roe"),
                                             ("line", "advection"),
                                             ("tile", "euler-hlle"),
                                             ("tile", "shallow-water-roe")])
def test_fused_cfl_epilogue_bitwise(monkeypatch, kernel_env, name):
    # opt-in WS_FUSE=1: the next step's CFL maxima come from the update
    # kernel's epilogue (+ tile-border pass) instead of the pre-pass; every dt
    # and the state must not change
    monkeypatch.setenv("WS_FUSE", "1")
    monkeypatch.setenv("WS_KERNEL", kernel_env)
    for bc in ("periodic", "extrapolate"):
        _compare(name, 131, 75, 5, 2, "mc", (bc, bc), seed=19)
        _compare(name, 131, 75, 5, 2, "superbee", (bc, bc), seed=20, use_run=True)


def test_fp32_c5_recipe_within_stated_bound():
    # configs[4] (C5) recipe at 256^2, 20 steps, MC: fp32 device vs the fp64
    # device run (itself bitwise the oracle) — the stated fp32 bound
    from paper_1308_1464_b200 import configs
    c = configs.c5_bumps(256, steps=20)
    q64, r64, _ = device_run(c.kernel, c.q, None, c.nx, c.ny, c.dx, c.dy, steps=20, order=2,
                             limiter="mc")
    q32, r32, _ = device_run(c.kernel, np.asfortranarray(c.q, dtype=np.float32), None, c.nx,
                             c.ny, c.dx, c.dy, steps=20, order=2, limiter="mc",
                             precision="f32")
    assert r64.error.code == 0 and r32.error.code == 0
    h64 = q64[0, 2:-2, 2:-2]
    h32 = q32[0, 2:-2, 2:-2].astype(np.float64)
    rel = np.abs(h32 - h64).max() / np.abs(h64).max()
    dts64 = np.array([r[0] for r in r64.reports])
    dts32 = np.array([r[0] for r in r32.reports])
    print(f"C5 recipe 256^2 x 20: fp32 max rel err on h {rel:.3e}, "
          f"max rel dt diff {np.abs(dts32 / dts64 - 1).max():.3e}")
    assert rel <= 1e-5, rel
    assert np.abs(dts32 / dts64 - 1).max() <= 1e-5


@pytest.mark.parametrize("name,bc", [("euler-hlle", "periodic"), ("euler", "extrapolate")])
def test_persistent_line_kernel_walks_tiles_bitwise(name, bc):
    # 4-component fp64 systems on 10-warp CTAs, two per SM: 264 tiles, more
    # than one per SM (the WS_GAS2=0 build: persistent 15-warp CTAs that walk
    # the tiles, prefetching the next with cp.async)
    _compare(name, 610, 331, 3, 2, "mc", (bc, bc), seed=23)


@pytest.mark.parametrize("name,order,limiter", [("shallow-water-roe", 2, "mc"),
                                                ("euler-hlle", 2, "minmod"),
                                                ("acoustics-var", 1, "none")])
def test_run_to_t_final_matches_oracle(name, order, limiter):
    # device-resident run with the t_final truncation decided on the GPU
    # (remaining = t_final - t, tolerance 1e-14 max(1, t_final), reference
    # driver.py:228-250): same number of steps, same dts (the last one
    # truncated), same state; the graph path is used (> 4 steps)
    from paper_1308_1464_b200 import _abi
    from helpers import device_grid
    nx, ny = 48, 37
    dx, dy = 1.0 / nx, 1.0 / ny
    q, aux = random_state(name, nx, ny, 24)
    oq = np.asfortranarray(q.copy())
    oa = np.asfortranarray(aux.copy()) if aux is not None else None
    solver = O.make_solver(name, **PARAMS[name])
    spec = O.Spec(nx, ny, dx, dy)
    probe = O.step(np.asfortranarray(q.copy()), oa, spec, solver, O.Controller(0.9),
                   bc_x="periodic", bc_y="periodic", order=order, limiter=limiter)
    t_final = 11.37 * probe.dt                 # ~12 steps, the last one truncated
    oreps = O.run(oq, oa, spec, solver, O.Controller(0.9), t_final=t_final,
                  bc_x="periodic", bc_y="periodic", order=order, limiter=limiter)
    g = device_grid(name, nx, ny, dx, dy, order=order, limiter=limiter, bc_x="periodic",
                    bc_y="periodic")
    try:
        g.upload(q, aux)
        g.run(50, _abi.make_ctl(0.9, t_final=t_final))   # more than needed: stops itself
        res = g.poll()
        assert res.error.code == 0
        assert res.steps_done == len(oreps)
        assert [r[0] for r in res.reports] == [r.dt for r in oreps]
        assert abs(res.t - t_final) <= 1e-14 * max(1.0, t_final)
        assert same_bits(oq, g.download())
    finally:
        g.close()


@pytest.mark.parametrize("first_steps,second", [(50, "t_final"), (50, "steps"), (3, "t_final")])
def test_t_final_runs_back_to_back_without_polling(first_steps, second):
    # a t_final run that stops early leaves the host's step count
    # ahead of the device's; the next run (larger t_final, or plain steps)
    # must continue from the newest state, not the stale ping-pong buffer
    from paper_1308_1464_b200 import _abi
    from helpers import device_grid
    name, nx, ny = "shallow-water-roe", 48, 37
    dx, dy = 1.0 / nx, 1.0 / ny
    q, aux = random_state(name, nx, ny, 31)
    solver = O.make_solver(name, **PARAMS[name])
    spec = O.Spec(nx, ny, dx, dy)
    kw = dict(bc_x="periodic", bc_y="periodic", order=2, limiter="mc")
    probe = O.step(np.asfortranarray(q.copy()), None, spec, solver, O.Controller(0.9), **kw)
    t1, t2 = 6.37 * probe.dt, 11.71 * probe.dt      # 7 steps (odd) then more
    oq = np.asfortranarray(q.copy())
    oreps = O.run(oq, None, spec, solver, O.Controller(0.9), t_final=t1, **kw)
    if second == "t_final":
        # the reference loop restarted with remaining = t2 - t
        t = sum(r.dt for r in oreps)
        while t2 - t > 1e-14 * max(1.0, t2):
            r = O.step(oq, None, spec, solver, O.Controller(0.9), remaining=t2 - t, **kw)
            oreps.append(r)
            t += r.dt
    else:
        oreps += [O.step(oq, None, spec, solver, O.Controller(0.9), **kw) for _ in range(4)]
    g = device_grid(name, nx, ny, dx, dy, **kw)
    try:
        g.upload(q, aux)
        g.run(first_steps, _abi.make_ctl(0.9, t_final=t1))   # stops itself after 7
        if first_steps < 7:
            g.run(50, _abi.make_ctl(0.9, t_final=t1))        # same t_final continues
        if second == "t_final":
            g.run(50, _abi.make_ctl(0.9, t_final=t2))
        else:
            g.run(4, _abi.make_ctl(0.9))
        res = g.poll()
        assert res.error.code == 0
        assert res.steps_done == len(oreps)
        assert [r[0] for r in res.reports] == [r.dt for r in oreps]
        assert same_bits(oq, g.download())
    finally:
        g.close()


def test_driver_run_t_final_and_remaining():
    # the public driver API: run(config with t_final) and step(remaining=...)
    from paper_1308_1464_b200 import (BoundaryCondition, GridSpec, SimulationConfig,
                                      TimestepController, initial_condition, run, step)
    spec = GridSpec(nx=40, ny=30, dx=1 / 40, dy=1 / 30, num_eqn=3, num_aux=0)
    cfg = SimulationConfig(spec=spec, kernel="shallow-water-roe", ic="sw-dam-break",
                           t_final=0.05, order=2, limiter="mc",
                           bc_x=BoundaryCondition.EXTRAPOLATE, bc_y=BoundaryCondition.EXTRAPOLATE)
    state, reps = run(cfg, TimestepController(0.9))
    assert abs(sum(r.dt for r in reps) - 0.05) <= 1e-14
    st, aux, _ = initial_condition("sw-dam-break", spec)
    oq = np.asfortranarray(st.data.copy())
    solver = O.make_solver("shallow-water-roe", **PARAMS["shallow-water-roe"])
    oreps = O.run(oq, None, O.Spec(40, 30, 1 / 40, 1 / 30), solver, O.Controller(0.9),
                  t_final=0.05, bc_x="extrapolate", bc_y="extrapolate", order=2, limiter="mc")
    assert [r.dt for r in reps] == [r.dt for r in oreps]
    assert same_bits(oq, state.data)
    # one step with remaining smaller than the CFL dt takes exactly `remaining`
    cfg1 = SimulationConfig(spec=spec, kernel="shallow-water-roe", ic="sw-dam-break",
                            num_steps=1, order=2, limiter="mc",
                            bc_x=BoundaryCondition.EXTRAPOLATE,
                            bc_y=BoundaryCondition.EXTRAPOLATE)
    st, aux, _ = initial_condition("sw-dam-break", spec)
    _, rep = step(st, aux, cfg1, TimestepController(0.9), remaining=1e-5)
    assert rep.dt == 1e-5


@pytest.mark.parametrize("env", ["WS_PDL=0", "WS_PERSIST=0", "WS_SPEEDS=smem", "WS_SPEEDS=exact",
                                 "WS_SPEEDS=edge"])
def test_alternative_launch_paths_bitwise(monkeypatch, env):
    # the non-default execution paths (plain launches, non-persistent 4-component
    # line kernel, shared-memory pre-pass) give the same bits
    k, v = env.split("=")
    monkeypatch.setenv(k, v)
    for name in ("shallow-water-roe", "euler-hlle", "acoustics-var"):
        _compare(name, 610, 97, 3, 2, "mc", ("periodic", "extrapolate"), seed=25)
    _compare("euler", 131, 75, 4, 2, "superbee", ("extrapolate", "extrapolate"), seed=26,
             use_run=True)
