"""ws_run on small static-speed grids: k_run_small runs every step in one
cooperative launch (one CTA per tile, a grid barrier per step, the step
records written by a control warp).  Bitwise equal to the oracle (state and
every dt) and to the per-step graph path (WS_RUN_SMALL=0), including
t_final / dt_max / fixed_dt controls and the error records."""

import os

import numpy as np
import pytest

from helpers import PARAMS, oracle_run, random_state
from oracle import wavestep_oracle as O

pytestmark = pytest.mark.gpu


def dev_run(name, q, aux, nx, ny, steps, *, order, limiter, bc, ctl, small=True, params=None):
    from paper_1308_1464_b200 import DeviceGrid, make_kernel
    old = os.environ.get("WS_RUN_SMALL")
    os.environ["WS_RUN_SMALL"] = "1" if small else "0"
    try:
        g = DeviceGrid(nx, ny, 1.0 / nx, 1.0 / ny, make_kernel(name, **(params or PARAMS[name])),
                       order=order, limiter=limiter, bc_x=bc, bc_y=bc)
    finally:
        if old is None:
            del os.environ["WS_RUN_SMALL"]
        else:
            os.environ["WS_RUN_SMALL"] = old
    try:
        g.upload(q, aux)
        l0 = g.launches()
        g.run(steps, ctl)
        launches = g.launches() - l0
        res = g.poll()
        out = g.download()
        return out, res, launches
    finally:
        g.close()


CASES = [("acoustics-const", 37, 29, "extrapolate", 2, "mc"),
         ("acoustics-const", 256, 256, "extrapolate", 2, "mc"),
         ("acoustics-const", 131, 75, "periodic", 2, "superbee"),
         ("acoustics-const", 300, 310, "periodic", 1, "none"),
         ("acoustics-var", 64, 97, "extrapolate", 2, "minmod"),
         ("acoustics-var", 200, 150, "periodic", 2, "mc"),
         ("advection", 90, 61, "periodic", 2, "mc"),
         ("advection", 5, 3, "extrapolate", 2, "mc")]


@pytest.mark.parametrize("name,nx,ny,bc,order,limiter", CASES)
def test_run_small_bitwise_vs_oracle_and_graph_path(name, nx, ny, bc, order, limiter):
    from paper_1308_1464_b200 import _abi
    steps = 13
    q, aux = random_state(name, nx, ny, 51)
    ref, oreps = oracle_run(name, q, aux, nx, ny, 1 / nx, 1 / ny, steps=steps, order=order,
                            limiter=limiter, bc_x=bc, bc_y=bc)
    ctl = _abi.make_ctl(0.9)
    out, res, launches = dev_run(name, q, aux, nx, ny, steps, order=order, limiter=limiter,
                                 bc=bc, ctl=ctl)
    assert launches == 1, "one cooperative launch for all steps"
    assert res.error.code == 0
    assert res.steps_done == steps
    assert [r[0] for r in res.reports] == [o.dt for o in oreps]
    assert [r[1] for r in res.reports] == [o.cfl for o in oreps]
    assert np.array_equal(out, ref)
    out2, res2, launches2 = dev_run(name, q, aux, nx, ny, steps, order=order, limiter=limiter,
                                    bc=bc, ctl=ctl, small=False)
    assert launches2 >= steps
    assert np.array_equal(out2, out) and res2.reports == res.reports and res2.t == res.t


@pytest.mark.parametrize("kw", [dict(t_final=7.3), dict(dt_max=0.6), dict(fixed_dt=0.45),
                                dict(t_final=3.0, dt_max=0.7)])
def test_run_small_controls_match_graph_path(kw):
    # t_final ends the run early inside the kernel (skip + finished); the
    # values are multiples of the CFL dt of this grid (dt ~ 0.0017 * scale)
    from paper_1308_1464_b200 import _abi
    name, nx, ny = "acoustics-const", 120, 88
    q, aux = random_state(name, nx, ny, 52)
    probe = O.step(np.asfortranarray(q.copy()), None, O.Spec(nx, ny, 1 / nx, 1 / ny),
                   O.make_solver(name, **PARAMS[name]), O.Controller(0.9), bc_x="periodic",
                   bc_y="periodic", order=2, limiter="mc")
    kw = {k: v * probe.dt for k, v in kw.items()}
    ctl = _abi.make_ctl(0.9, kw.get("dt_max"), kw.get("fixed_dt"), None, kw.get("t_final"))
    a = dev_run(name, q, aux, nx, ny, 20, order=2, limiter="mc", bc="periodic", ctl=ctl)
    b = dev_run(name, q, aux, nx, ny, 20, order=2, limiter="mc", bc="periodic", ctl=ctl,
                small=False)
    assert a[2] == 1
    assert a[1].steps_done == b[1].steps_done
    assert a[1].reports == b[1].reports and a[1].t == b[1].t
    assert a[1].error.code == b[1].error.code == 0
    assert np.array_equal(a[0], b[0])
    if "t_final" in kw:
        assert a[1].steps_done < 20
        assert abs(a[1].t - kw["t_final"]) <= 1e-14 * max(1.0, kw["t_final"])


def test_run_small_inadmissible_and_stationary_records():
    from paper_1308_1464_b200 import _abi
    # acoustics-var with a non-positive density in one cell: the first step's
    # checked probes report it (reference location), nothing is committed
    name, nx, ny = "acoustics-var", 70, 45
    q, aux = random_state(name, nx, ny, 53)
    aux[0, 2 + 33, 2 + 20] = -1.0
    ctl = _abi.make_ctl(0.9)
    a = dev_run(name, q, aux, nx, ny, 8, order=2, limiter="mc", bc="extrapolate", ctl=ctl)
    b = dev_run(name, q, aux, nx, ny, 8, order=2, limiter="mc", bc="extrapolate", ctl=ctl,
                small=False)
    assert a[1].error.code == _abi.WS_ERR_KERNEL
    for f in ("code", "direction", "i", "j", "stage", "component", "step"):
        assert getattr(a[1].error, f) == getattr(b[1].error, f), f
    assert a[1].steps_done == b[1].steps_done == 0
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[0][:, 2:-2, 2:-2], q[:, 2:-2, 2:-2])
    # advection at rest: every rate is zero -> the stationary record
    name = "advection"
    q, _ = random_state(name, 40, 30, 54)
    kw = dict(order=2, limiter="mc", bc="periodic", ctl=ctl, params={"u": 0.0, "v": 0.0})
    a = dev_run(name, q, None, 40, 30, 6, **kw)
    b = dev_run(name, q, None, 40, 30, 6, small=False, **kw)
    assert a[1].error.code == b[1].error.code == _abi.WS_ERR_STATIONARY
    assert a[1].steps_done == b[1].steps_done == 0


def test_run_small_back_to_back_runs_and_steps():
    # runs of the multi-step kernel mixed with single steps continue from the
    # newest state (odd step counts flip the ping-pong parity)
    from paper_1308_1464_b200 import _abi, DeviceGrid, make_kernel
    name, nx, ny = "acoustics-const", 96, 80
    q, aux = random_state(name, nx, ny, 55)
    ref, oreps = oracle_run(name, q, aux, nx, ny, 1 / nx, 1 / ny, steps=5 + 1 + 7 + 4,
                            order=2, limiter="mc", bc_x="periodic", bc_y="periodic")
    g = DeviceGrid(nx, ny, 1 / nx, 1 / ny, make_kernel(name, **PARAMS[name]), order=2,
                   limiter="mc", bc_x="periodic", bc_y="periodic")
    try:
        g.upload(q, aux)
        ctl = _abi.make_ctl(0.9)
        g.run(5, ctl)
        g.step(ctl)
        g.run(7, ctl)
        g.run(4, ctl)
        res = g.poll()
        assert res.error.code == 0
        assert [r[0] for r in res.reports] == [o.dt for o in oreps]
        assert np.array_equal(g.download(), ref)
    finally:
        g.close()


def test_step_inside_a_caller_capture_uses_the_per_step_kernels():
    # ws_step on a small static-speed grid is one k_run_small launch, except
    # inside a caller's stream capture (a cooperative launch there could
    # invalidate it): the captured graph replays bitwise
    import torch
    from paper_1308_1464_b200 import DeviceGrid, _abi, make_kernel
    name, nx, ny = "acoustics-const", 64, 48
    q, aux = random_state(name, nx, ny, 56)
    ref, oreps = oracle_run(name, q, aux, nx, ny, 1 / nx, 1 / ny, steps=8, order=2,
                            limiter="mc", bc_x="periodic", bc_y="periodic")
    g = DeviceGrid(nx, ny, 1 / nx, 1 / ny, make_kernel(name, **PARAMS[name]), order=2,
                   limiter="mc", bc_x="periodic", bc_y="periodic")
    try:
        s = torch.cuda.Stream()
        g.upload(q, aux, stream=s.cuda_stream)
        ctl = _abi.make_ctl(0.9)
        g.step(ctl, stream=s.cuda_stream)
        g.step(ctl, stream=s.cuda_stream)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        g.capture_begin()
        with torch.cuda.graph(graph, stream=s):
            g.step(ctl, stream=s.cuda_stream)
            g.step(ctl, stream=s.cuda_stream)
        steps, launches = g.capture_end()
        assert steps == 2 and launches == 2          # the per-step update kernels
        for _ in range(3):
            with torch.cuda.stream(s):
                graph.replay()
            g.replayed(steps, launches)
        torch.cuda.synchronize()
        res = g.poll()
        assert res.error.code == 0 and res.steps_done == 8
        assert [r[0] for r in res.reports] == [o.dt for o in oreps]
        assert np.array_equal(g.download(stream=s.cuda_stream), ref)
    finally:
        g.close()
