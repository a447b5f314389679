"""Parity at BASELINE.json's full sizes on the B200.

* C2 (configs[1]) exactly as specified — 1024^2 shallow water, MC, CFL 0.9,
  200 steps — against the numpy oracle on every host core: identical state
  (np.array_equal) and all 200 dts identical.
* Size-independent properties where the oracle cannot follow in seconds:
  mass conservation with periodic BCs on the C5 recipe at 4096^2, and the
  1-GPU result of C3 (4096^2 Euler-HLLE) through two independent device
  paths (per-step calls vs the graph-replayed run) — bitwise.
"""

import os

import numpy as np
import pytest

from helpers import device_run, oracle_run

pytestmark = pytest.mark.gpu


def test_c2_full_size_200_steps_bitwise_vs_oracle():
    from paper_1308_1464_b200 import configs
    c = configs.c2_shallow_water()
    assert (c.nx, c.ny, c.steps) == (1024, 1024, 200)
    dq, res, _ = device_run(c.kernel, c.q, None, c.nx, c.ny, c.dx, c.dy, steps=c.steps,
                            order=2, limiter="mc", bc_x="extrapolate", bc_y="extrapolate",
                            use_run=True)
    oq, oreps = oracle_run(c.kernel, c.q, None, c.nx, c.ny, c.dx, c.dy, steps=c.steps,
                           order=2, limiter="mc", bc_x="extrapolate", bc_y="extrapolate",
                           threads=os.cpu_count() or 1)
    assert res.error.code == 0 and res.steps_done == 200
    assert [r[0] for r in res.reports] == [r.dt for r in oreps]
    assert np.array_equal(dq, oq)


def test_periodic_mass_conservation_at_4096():
    # C5 recipe (64 Gaussian bumps) at 4096^2, periodic, 20 MC steps: the
    # flux-difference form conserves sum(h) up to rounding
    from paper_1308_1464_b200 import configs
    c = configs.c5_bumps(4096, steps=20)
    dq, res, _ = device_run(c.kernel, c.q, None, c.nx, c.ny, c.dx, c.dy, steps=20, order=2,
                            limiter="mc", bc_x="periodic", bc_y="periodic", use_run=True)
    assert res.error.code == 0
    m0 = np.sum(c.q[0, 2:-2, 2:-2], dtype=np.float64)
    m1 = np.sum(dq[0, 2:-2, 2:-2], dtype=np.float64)
    assert abs(m1 - m0) <= 1e-12 * abs(m0), (m0, m1)


def test_c3_full_size_step_calls_equal_graph_run():
    from paper_1308_1464_b200 import configs
    c = configs.c3_euler_quadrants()
    assert (c.nx, c.ny) == (4096, 4096)
    a, ra, _ = device_run(c.kernel, c.q, None, c.nx, c.ny, c.dx, c.dy, steps=10, order=2,
                          limiter="minmod", cfl=c.cfl, use_run=True)
    b, rb, _ = device_run(c.kernel, c.q, None, c.nx, c.ny, c.dx, c.dy, steps=10, order=2,
                          limiter="minmod", cfl=c.cfl, use_run=False)
    assert ra.error.code == 0 and rb.error.code == 0
    assert [r[0] for r in ra.reports] == [r[0] for r in rb.reports]
    assert np.array_equal(a, b)
