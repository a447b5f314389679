"""Wide, short grids on the B200: the line kernel's L2 band prefetch splits a
halo row into several segments once a tile row has more CTAs than the band
has row-components (ntx >= 33 * (num_eqn + num_aux): 3 components from 2871
cells across, 4 from 3828, 5 from 4785; two segments from twice that), and
looks `ceil(444 / ntx)` tile rows ahead.  The prefetch is only a hint, so
the check is the usual one — state and every dt bitwise equal to the oracle
— on shapes that drive those branches: multi-segment rows for every
component count, partial last tiles in x and y, both boundary conditions,
fp64 and fp32.
"""

import numpy as np
import pytest

from helpers import device_run, oracle_run, random_state

pytestmark = pytest.mark.gpu

CASES = [
    # kernel, nx, ny, limiter, bc
    ("acoustics-var", 9600, 64, "mc", "extrapolate"),       # 5 components, ntx = 332: two segments
    ("shallow-water-roe", 5800, 45, "mc", "periodic"),      # 3 components, ntx = 200: two segments
    ("euler-hlle", 7700, 31, "minmod", "extrapolate"),      # 4 components, ntx = 266: two segments
    ("acoustics-var", 4790, 90, "superbee", "periodic"),    # ntx = 166 >= 165: one segment, 3 rows ahead
]


@pytest.mark.parametrize("name,nx,ny,limiter,bc", CASES)
def test_wide_grid_bitwise_vs_oracle(name, nx, ny, limiter, bc):
    q, aux = random_state(name, nx, ny, seed=nx + ny)
    dx, dy = 1.0 / nx, 1.0 / ny
    kw = dict(steps=3, order=2, limiter=limiter, bc_x=bc, bc_y=bc)
    dq, res, _ = device_run(name, q, aux, nx, ny, dx, dy, **kw)
    oq, oreps = oracle_run(name, q, aux, nx, ny, dx, dy, threads=8, **kw)
    assert res.error.code == 0 and res.steps_done == 3
    assert [r[0] for r in res.reports] == [r.dt for r in oreps]
    assert np.array_equal(dq, oq)


def test_wide_grid_fp32_bitwise_vs_fp32_oracle():
    # fp32 interior tiles go through stage_inner (LinePolicy::FASTSTAGE)
    name, nx, ny = "shallow-water-roe", 5800, 45
    q, aux = random_state(name, nx, ny, seed=7, dtype=np.float32)
    dx, dy = 1.0 / nx, 1.0 / ny
    oq, oreps = oracle_run(name, q, aux, nx, ny, dx, dy, steps=3, order=2, limiter="mc", threads=8)
    assert oq.dtype == np.float32
    dq, res, _ = device_run(name, q, aux, nx, ny, dx, dy, steps=3, order=2, limiter="mc",
                            precision="f32")
    assert res.error.code == 0
    assert [r.dt for r in oreps] == [r[0] for r in res.reports]
    assert np.array_equal(oq, dq)
