"""Parity on every BASELINE.json recipe (configs[0..4]).

north_star: the device step must match the reference's step on identical
seeded inputs, and the CFL dt must be identical.  Each recipe runs on the
B200 through the C ABI and in the numpy oracle on every host core, from the
same input bytes (paper_1308_1464_b200.configs); the whole state (ghost
frame included) must be bitwise equal and every step's dt, cfl and max
speeds identical (tolerance: zero).  Reference anchors: the step
driver.py:199-225, the bitwise twin guard bench.py:181-185.

* C1 exactly as specified: 256^2 const acoustics, MC, CFL 0.9, 100 steps.
* C2 exactly as specified: test_gpu_fullsize.py (1024^2, 200 steps).
* C3 at its full 4096^2 (Euler HLLE, minmod, CFL 0.8) for 10 of its 50 steps.
* C4 at its full 8192^2 (lognormal var acoustics, MC) for 5 steps, and the
  same recipe at 2048^2 for 50 steps (its full step count).
* C5 fp64 (64 bumps, SW Roe + Harten, MC): the recipe at 4096^2 for its 20
  steps.
* C5 fp32 against C5 fp64 on the device at the full 16384^2 x 20 steps:
  stated bound rel max|dh| / max|h| <= 1e-5 and every dt within 1e-5
  (DESIGN.md §6); fp32 is also bitwise equal to an fp32 oracle run of the
  recipe at 1024^2 x 20.
"""

import numpy as np
import pytest

from helpers import assert_same_run, case_device_run, case_oracle_run

pytestmark = pytest.mark.gpu


def _check(case, steps):
    dq, res = case_device_run(case, steps)
    oq, oreps = case_oracle_run(case, steps)
    assert_same_run(oq, oreps, dq, res, steps)
    return oreps


def test_c1_as_specified_mc_100_steps():
    from paper_1308_1464_b200 import configs
    c = configs.c1_acoustics()
    assert (c.nx, c.ny, c.limiter, c.order, c.cfl, c.steps) == (256, 256, "mc", 2, 0.9, 100)
    assert c.kernel_params == {"rho": 1.0, "bulk": 4.0}
    oreps = _check(c, 100)
    # constant speeds c = 2: dt = 0.9 / (2/dx + 2/dy) = 0.9/1024 every step
    assert all(r.dt == 0.9 / 1024.0 for r in oreps)


def test_c3_full_size_10_steps():
    from paper_1308_1464_b200 import configs
    c = configs.c3_euler_quadrants()
    assert (c.nx, c.ny, c.limiter, c.cfl) == (4096, 4096, "minmod", 0.8)
    _check(c, 10)


def test_c4_full_size_5_steps():
    from paper_1308_1464_b200 import configs
    c = configs.c4_var_acoustics()
    assert (c.nx, c.ny, c.limiter) == (8192, 8192, "mc")
    _check(c, 5)


def test_c4_recipe_2048_all_50_steps():
    from paper_1308_1464_b200 import configs
    c = configs.c4_var_acoustics(2048)
    _check(c, 50)


def test_c5_fp64_recipe_4096_20_steps():
    from paper_1308_1464_b200 import configs
    c = configs.c5_bumps(4096)
    assert (c.limiter, c.cfl, c.steps) == ("mc", 0.9, 20)
    _check(c, 20)


def test_c5_device_generator_has_the_host_bits():
    # bench.py builds the 16384^2 field on the GPU: it must be the recipe's
    # host field bit for bit (both arms of the bench see the same input)
    import torch
    from paper_1308_1464_b200 import configs
    host = configs.c5_bumps(2048)
    dev = configs.c5_bumps(2048, device=torch.device("cuda", 0))
    h = dev.meta["h_dev"].t().contiguous().cpu().numpy()
    assert np.array_equal(host.q[0, 2:-2, 2:-2], h)
    band = configs.c5_bumps(2048, rows=(700, 900))
    assert np.array_equal(band.q[0, 2:-2, 2:-2], h[:, 700:900])


def test_c5_fp32_bitwise_vs_fp32_oracle_1024():
    from paper_1308_1464_b200 import configs
    c = configs.c5_bumps(1024)
    dq, res = case_device_run(c, 20, precision="f32")
    oq, oreps = case_oracle_run(c, 20, dtype=np.float32)
    assert_same_run(oq, oreps, dq, res, 20)


def test_c5_fp32_vs_fp64_full_size_within_stated_bound():
    # the full 16384^2 x 20 recipe on the device in both precisions
    from paper_1308_1464_b200 import configs
    import torch
    c = configs.c5_bumps(16384, device=torch.device("cuda", 0))
    h = c.meta.pop("h_dev").t().contiguous().cpu().numpy()
    q = configs._field(3, c.nx, c.ny)
    q[0, 2:-2, 2:-2] = h
    del h
    c.q = q
    d64, r64 = case_device_run(c, 20, precision="f64")
    d32, r32 = case_device_run(c, 20, precision="f32")
    assert r64.error.code == 0 and r32.error.code == 0
    assert r64.steps_done == r32.steps_done == 20
    h64 = d64[0, 2:-2, 2:-2]
    rel = float(np.abs(d32[0, 2:-2, 2:-2].astype(np.float64) - h64).max() / np.abs(h64).max())
    assert rel <= 1e-5, rel
    dts64 = np.array([r[0] for r in r64.reports])
    dts32 = np.array([r[0] for r in r32.reports])
    assert np.abs(dts32 / dts64 - 1.0).max() <= 1e-5
