"""The fp32 throughput mode (precision "f32fast", WS_FP32_FAST): the same
kernels compiled with FMA contraction and the approximate MUFU division /
square root.  Its parity is the stated bound against fp64 -- max relative
error <= 1e-5 on every state component (max |q32 - q64| / max |q64|) and on
every dt after 20 steps -- not bits; the CFL pre-pass filter stays exact
against its own probes (tile pre-pass == probing every edge, bitwise), and
inadmissible states are reported at the same interface as in fp64."""

import os

import numpy as np
import pytest

from helpers import PARAMS, case_device_run, oracle_run, random_state

pytestmark = pytest.mark.gpu
BOUND = 1e-5


def fast_run(name, q, aux, nx, ny, steps, *, order, limiter, bc, env=None):
    from paper_1308_1464_b200 import DeviceGrid, _abi, make_kernel
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        g = DeviceGrid(nx, ny, 1 / nx, 1 / ny, make_kernel(name, **PARAMS[name]), order=order,
                       limiter=limiter, bc_x=bc, bc_y=bc, precision="f32fast")
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
    try:
        g.upload(np.asfortranarray(q, dtype=np.float32),
                 np.asfortranarray(aux, dtype=np.float32) if aux is not None else None)
        g.run(steps, _abi.make_ctl(0.9))
        res = g.poll()
        return g.download(), res
    finally:
        g.close()


def rel_err(q32, q64):
    """max over components of max |q32 - q64| / max |q64| (interior cells)."""
    a, b = q32[:, 2:-2, 2:-2].astype(np.float64), q64[:, 2:-2, 2:-2]
    return max(float(np.abs(a[c] - b[c]).max() / max(np.abs(b[c]).max(), 1e-300))
               for c in range(b.shape[0]))


@pytest.mark.parametrize("name,bc,order,limiter", [
    ("shallow-water-roe", "extrapolate", 2, "mc"), ("shallow-water-roe", "periodic", 2, "superbee"),
    ("euler-hlle", "periodic", 2, "minmod"), ("euler", "extrapolate", 2, "mc"),
    ("acoustics-const", "periodic", 2, "mc"), ("acoustics-var", "extrapolate", 2, "mc"),
    ("advection", "periodic", 2, "mc"), ("euler", "periodic", 1, "none")])
def test_fast_fp32_within_stated_bound_of_the_fp64_oracle(name, bc, order, limiter):
    nx, ny, steps = 96, 71, 20
    q, aux = random_state(name, nx, ny, 61)
    ref, oreps = oracle_run(name, q, aux, nx, ny, 1 / nx, 1 / ny, steps=steps, order=order,
                            limiter=limiter, bc_x=bc, bc_y=bc)
    out, res = fast_run(name, q, aux, nx, ny, steps, order=order, limiter=limiter, bc=bc)
    assert res.error.code == 0 and res.steps_done == steps
    err = rel_err(out, ref)
    dts = np.array([r[0] for r in res.reports])
    odts = np.array([o.dt for o in oreps])
    print(f"{name} {bc} o{order} {limiter}: state rel {err:.2e}, dt rel "
          f"{np.abs(dts / odts - 1).max():.2e}")
    assert err <= BOUND, err
    assert np.abs(dts / odts - 1).max() <= BOUND


@pytest.mark.parametrize("name", ["shallow-water-roe", "euler-hlle"])
def test_fast_fp32_tile_prepass_equals_probing_every_edge(name):
    # the tile filter's bound argument holds for the fast arithmetic too: the
    # default run and the WS_SPEEDS=exact run are bitwise the same
    nx, ny, steps = 300, 200, 12
    q, aux = random_state(name, nx, ny, 62)
    a = fast_run(name, q, aux, nx, ny, steps, order=2, limiter="mc", bc="extrapolate")
    b = fast_run(name, q, aux, nx, ny, steps, order=2, limiter="mc", bc="extrapolate",
                 env={"WS_SPEEDS": "exact"})
    assert a[1].error.code == b[1].error.code == 0
    assert a[1].reports == b[1].reports
    assert np.array_equal(a[0], b[0])


def test_fast_fp32_reports_the_fp64_error_location():
    from paper_1308_1464_b200 import _abi
    from helpers import device_run
    name, nx, ny = "shallow-water-roe", 70, 45
    q, _ = random_state(name, nx, ny, 63)
    q[0, 2 + 40, 2 + 17] = -0.5
    out, res = fast_run(name, q, None, nx, ny, 3, order=2, limiter="mc", bc="extrapolate")
    _, r64, _ = device_run(name, q, None, nx, ny, 1 / nx, 1 / ny, steps=3, order=2,
                           limiter="mc", use_run=True)
    assert res.error.code == r64.error.code == _abi.WS_ERR_KERNEL
    for f in ("direction", "i", "j", "stage", "component", "step"):
        assert getattr(res.error, f) == getattr(r64.error, f), f


def test_fast_fp32_c5_full_size_within_stated_bound():
    # the 16384^2 x 20 recipe on the device, fast fp32 against fp64
    from paper_1308_1464_b200 import configs
    import torch
    c = configs.c5_bumps(16384, device=torch.device("cuda", 0))
    h = c.meta.pop("h_dev").t().contiguous().cpu().numpy()
    q = configs._field(3, c.nx, c.ny)
    q[0, 2:-2, 2:-2] = h
    del h
    c.q = q
    d64, r64 = case_device_run(c, 20, precision="f64")
    d32, r32 = case_device_run(c, 20, precision="f32fast")
    assert r64.error.code == 0 and r32.error.code == 0
    assert r64.steps_done == r32.steps_done == 20
    h64 = d64[0, 2:-2, 2:-2]
    rel = float(np.abs(d32[0, 2:-2, 2:-2].astype(np.float64) - h64).max() / np.abs(h64).max())
    dts64 = np.array([r[0] for r in r64.reports])
    dts32 = np.array([r[0] for r in r32.reports])
    print(f"C5 16384^2 x 20 fast fp32: h rel {rel:.2e}, dt rel {np.abs(dts32 / dts64 - 1).max():.2e}")
    assert rel <= BOUND, rel
    assert np.abs(dts32 / dts64 - 1).max() <= BOUND
