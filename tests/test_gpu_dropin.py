"""The reference-shaped drop-in surface on the GPU: fill_ghost and driver.step.

* ``grid.fill_ghost`` (C ABI ws_fill_ghost) equals the reference's own
  fill_ghost (grid.py:179-193) on the committed golden vectors
  (tests/golden/fill_ghost_golden.json, made by running the reference):
  both BCs, mixed pairs, corners, n == num_ghost.
* ``driver.step`` mutates its arguments the way the reference's step does
  (driver.py:199-225): the state comes back advanced with its ghost frame
  filled from the state the step started from, and the aux ghost frame is
  refilled every step (driver.py:211-212); on an inadmissible state the
  SweepError is raised after those ghost fills, interior untouched.
* the caller's arrays are page-locked once (ws_pin_host) and reused.
"""

import json
import os

import numpy as np
import pytest

from helpers import PARAMS, random_state
from oracle import wavestep_oracle as O

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
FILL = json.load(open(os.path.join(HERE, "golden", "fill_ghost_golden.json")))


@pytest.mark.parametrize("k", range(len(FILL["cases"])))
def test_fill_ghost_on_device_matches_reference_golden(k):
    from paper_1308_1464_b200 import BoundaryCondition, GridSpec, StateField, fill_ghost
    c = FILL["cases"][k]
    shape = (c["ncomp"], c["nx"] + 4, c["ny"] + 4)
    before = np.array(c["before"]).reshape(shape, order="F")
    after = np.array(c["after"]).reshape(shape, order="F")
    spec = GridSpec(nx=c["nx"], ny=c["ny"], dx=1.0 / c["nx"], dy=1.0 / c["ny"],
                    num_eqn=c["ncomp"], num_aux=0)
    f = StateField(spec)
    f.data[...] = before
    out = fill_ghost(f, BoundaryCondition(c["bc_x"]), BoundaryCondition(c["bc_y"]))
    assert out is f
    assert np.array_equal(f.data, after)


def _setup(name, nx, ny, bc, seed, order=1, limiter="none"):
    from paper_1308_1464_b200 import (AuxField, BoundaryCondition, GridSpec,
                                      SimulationConfig, StateField)
    from paper_1308_1464_b200.kernels import DESCRIPTORS
    d = DESCRIPTORS[name]
    spec = GridSpec(nx=nx, ny=ny, dx=1.0 / nx, dy=1.0 / ny, num_eqn=d.num_eqn,
                    num_aux=d.num_aux)
    q, aux = random_state(name, nx, ny, seed)
    st, ax = StateField(spec), AuxField(spec)
    st.data[...] = q
    st.data[:, :2, :] = 7.0          # stale ghost garbage the step must overwrite
    if aux is not None:
        ax.data[...] = aux
        ax.data[:, :, -2:] = -3.0
    cfg = SimulationConfig(spec=spec, kernel=name, ic="x", num_steps=1, order=order,
                           limiter=limiter, bc_x=BoundaryCondition(bc), bc_y=BoundaryCondition(bc),
                           kernel_params=PARAMS[name])
    return spec, st, ax, cfg


@pytest.mark.parametrize("name,bc,order", [("acoustics-var", "extrapolate", 1),
                                           ("acoustics-var", "periodic", 2),
                                           ("shallow-water-roe", "periodic", 2),
                                           ("euler", "extrapolate", 1)])
def test_driver_step_mutates_state_and_aux_like_the_reference(name, bc, order):
    from paper_1308_1464_b200 import TimestepController, step
    lim = "mc" if order == 2 else "none"
    spec, st, ax, cfg = _setup(name, 300, 280, bc, 41, order, lim)
    oq = np.asfortranarray(st.data.copy())
    oa = np.asfortranarray(ax.data.copy()) if spec.num_aux else None
    solver = O.make_solver(name, **PARAMS[name])
    ospec = O.Spec(spec.nx, spec.ny, spec.dx, spec.dy)
    for _ in range(3):
        orep = O.step(oq, oa, ospec, solver, O.Controller(0.9), bc_x=bc, bc_y=bc, order=order,
                      limiter=lim)
        _, rep = step(st, ax if spec.num_aux else None, cfg, TimestepController(0.9))
        assert (rep.dt, rep.max_speed_x, rep.max_speed_y) == (orep.dt, orep.max_speed_x,
                                                             orep.max_speed_y)
        assert np.array_equal(st.data, oq)              # whole array, ghost frame included
        if spec.num_aux:
            assert np.array_equal(ax.data, oa)          # aux ghosts refilled, interior kept


def test_driver_step_error_mutates_ghosts_then_raises():
    from paper_1308_1464_b200 import SweepError, TimestepController, step
    name = "acoustics-var"
    spec, st, ax, cfg = _setup(name, 40, 30, "extrapolate", 42)
    st.data[1, 2 + 5, 2 + 3] = np.nan
    q0 = st.data.copy(order="F")
    oq, oa = np.asfortranarray(q0.copy()), np.asfortranarray(ax.data.copy())
    with pytest.raises(O.OracleError) as oe:
        O.step(oq, oa, O.Spec(40, 30, 1 / 40, 1 / 30), O.make_solver(name), O.Controller(0.9),
               bc_x="extrapolate", bc_y="extrapolate")
    with pytest.raises(SweepError) as de:
        step(st, ax, cfg, TimestepController(0.9))
    assert str(de.value) == str(oe.value)
    # the oracle (like the reference) filled both ghost frames before raising
    assert np.array_equal(st.data, oq, equal_nan=True)
    assert np.array_equal(ax.data, oa)
    assert np.array_equal(st.data[:, 2:-2, 2:-2], q0[:, 2:-2, 2:-2], equal_nan=True)


def test_driver_step_pins_the_callers_arrays_once():
    from paper_1308_1464_b200 import TimestepController, driver, step
    spec, st, ax, cfg = _setup("shallow-water-roe", 512, 512, "extrapolate", 43)
    step(st, None, cfg, TimestepController(0.9))
    key = (st.data.ctypes.data, st.data.nbytes)
    assert key in driver._PINNED and driver._PINNED[key][0]() is st.data
    n = len(driver._PINNED)
    step(st, None, cfg, TimestepController(0.9))
    assert len(driver._PINNED) == n
    data = st.data
    st.data = np.asfortranarray(data.copy())
    del data
    import gc
    gc.collect()
    assert key not in driver._PINNED         # released (ws_unpin_host) with the array
