"""Pin the CPU oracle to the reference (CPU only).

1. Against tests/golden/reference_golden.json, produced by running the
   reference wavesweep itself (tests/golden/make_golden.py): every dt and
   max speed equal, final-state hash equal (bitwise), error text equal,
   kernel outputs equal.
2. Live against the reference when /root/reference is present (the build
   container): randomized cases through wavesweep.driver.step.
"""

import hashlib
import json
import os
import shutil
import sys
import tempfile

import numpy as np
import pytest

from helpers import random_state
from oracle import wavestep_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "reference_golden.json")))


def state_hash(q):
    c = np.asfortranarray(q, dtype=np.float64) + 0.0
    return hashlib.sha256(c.tobytes(order="F")).hexdigest()


def _input(name, case):
    if name == "c1-full":
        from paper_1308_1464_b200 import configs
        c = configs.c1_acoustics()
        return c.q.copy(order="F"), None
    return random_state(case["kernel"], case["nx"], case["ny"], case["seed"])


@pytest.mark.parametrize("name", sorted(GOLD["steps"]))
def test_oracle_matches_reference_golden_steps(name):
    case = GOLD["steps"][name]
    q, aux = _input(name, case)
    q = np.asfortranarray(q)
    solver = O.make_solver(case["kernel"], **case["params"])
    spec = O.Spec(case["nx"], case["ny"], case["dx"], case["dy"])
    reps = [O.step(q, aux, spec, solver, O.Controller(0.9), bc_x=case["bc_x"],
                   bc_y=case["bc_y"]) for _ in range(case["steps"])]
    assert [r.dt for r in reps] == case["dts"]
    assert [r.max_speed_x for r in reps] == case["msx"]
    assert [r.max_speed_y for r in reps] == case["msy"]
    assert [r.cfl for r in reps] == case["cfl"]
    assert state_hash(q) == case["q_sha256"]


def test_c1_dt_is_the_constant_cfl_step():
    # config-1 inputs give constant dt = 0.9/1024
    assert set(GOLD["steps"]["c1-full"]["dts"]) == {0.9 / 1024}


@pytest.mark.parametrize("key", sorted(GOLD["kernels"]))
def test_oracle_kernels_match_reference(key):
    case = GOLD["kernels"][key]
    name, d = key.rsplit("-", 1)
    ni = 1 if d == "x" else 2
    solver = O.make_solver(name, **case["params"])
    al = np.array(case["auxl"]) if "auxl" in case else None
    ar = np.array(case["auxr"]) if "auxr" in case else None
    w, s, am, ap = solver.solve(ni, np.array(case["ql"]), np.array(case["qr"]), al, ar)
    assert np.array_equal(am, np.array(case["amdq"]))
    assert np.array_equal(ap, np.array(case["apdq"]))
    assert np.array_equal(s, np.array(case["speeds"]))
    assert np.array_equal(w, np.array(case["waves"]))


@pytest.mark.parametrize("key", sorted(GOLD["errors"]))
def test_oracle_error_text_matches_reference(key):
    case = GOLD["errors"][key]
    q, aux = random_state(case["kernel"], case["nx"], case["ny"], case["seed"])
    q[case["comp"], 2 + 5, 2 + 3] = float(eval(case["value"], {"nan": np.nan, "inf": np.inf}))
    solver = O.make_solver(case["kernel"], **case["params"])
    spec = O.Spec(case["nx"], case["ny"], 1 / case["nx"], 1 / case["ny"])
    with pytest.raises(O.OracleError) as e:
        O.step(q, aux, spec, solver, O.Controller(0.9))
    assert str(e.value) == case["message"]


# ---------------------------------------------------------------------------
# live reference (build container only)

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def W():
    if not os.path.isdir(REF):
        pytest.skip("reference not present (GPU box)")
    tmp = tempfile.mkdtemp()
    shutil.copytree(REF, os.path.join(tmp, "src"))
    sys.path.insert(0, os.path.join(tmp, "src"))
    import wavesweep
    import wavesweep.oracles  # noqa: F401
    return wavesweep


@pytest.mark.parametrize("seed", range(6))
def test_oracle_matches_live_reference_randomized(W, seed):
    rng = np.random.default_rng(100 + seed)
    kernel = ["acoustics-const", "acoustics-var", "euler"][seed % 3]
    params = {"acoustics-const": {"rho": 1.3, "bulk": 2.1}, "acoustics-var": {},
              "euler": {"gamma": 1.4}}[kernel]
    nx, ny = int(rng.integers(2, 40)), int(rng.integers(2, 40))
    bcx, bcy = rng.choice(["periodic", "extrapolate"], 2)
    q, aux = random_state(kernel, nx, ny, seed)
    d = W.DESCRIPTORS[kernel]
    spec = W.GridSpec(nx=nx, ny=ny, dx=1 / nx, dy=0.7 / ny, num_eqn=d.num_eqn,
                      num_aux=d.num_aux)
    st, ax = W.StateField(spec), W.AuxField(spec)
    st.data[...] = q
    if aux is not None:
        ax.data[...] = aux
    cfg = W.SimulationConfig(spec=spec, kernel=kernel, ic=W.DEFAULT_IC[kernel], num_steps=1,
                             bc_x=W.BoundaryCondition(bcx), bc_y=W.BoundaryCondition(bcy),
                             kernel_params=params)
    oq = np.asfortranarray(q.copy())
    solver = O.make_solver(kernel, **params)
    for _ in range(5):
        _, r = W.step(st, ax, cfg, W.TimestepController(0.8))
        o = O.step(oq, aux, O.Spec(nx, ny, 1 / nx, 0.7 / ny), solver, O.Controller(0.8),
                   bc_x=str(bcx), bc_y=str(bcy), threads=1 + seed % 3)
        assert (r.dt, r.max_speed_x, r.max_speed_y) == (o.dt, o.max_speed_x, o.max_speed_y)
    assert np.array_equal(st.data, oq)


def test_order2_without_limiter_reduces_to_reference(W):
    """Oracle extension constraint: order=2/limiter none == reference order 1."""
    q, _ = random_state("euler", 20, 17, 3)
    spec = W.GridSpec(nx=20, ny=17, dx=0.05, dy=0.05, num_eqn=4)
    st = W.StateField(spec)
    st.data[...] = q
    cfg = W.SimulationConfig(spec=spec, kernel="euler", ic="euler-sod-x", num_steps=1,
                             bc_x=W.BoundaryCondition.EXTRAPOLATE,
                             bc_y=W.BoundaryCondition.EXTRAPOLATE)
    oq = np.asfortranarray(q.copy())
    for _ in range(3):
        W.step(st, W.AuxField(spec), cfg, W.TimestepController(0.9))
        O.step(oq, None, O.Spec(20, 17, 0.05, 0.05), O.make_solver("euler"),
               O.Controller(0.9), order=2, limiter="none")
    assert np.array_equal(st.data, oq)


FILL = json.load(open(os.path.join(HERE, "golden", "fill_ghost_golden.json")))


def _fill_case(c):
    shape = (c["ncomp"], c["nx"] + 4, c["ny"] + 4)
    before = np.array(c["before"]).reshape(shape, order="F")
    after = np.array(c["after"]).reshape(shape, order="F")
    return before, after


@pytest.mark.parametrize("k", range(len(FILL["cases"])))
def test_oracle_fill_ghost_matches_reference_golden(k):
    # reference grid.py:179-193, both BCs, corners from the x-filled columns
    c = FILL["cases"][k]
    before, after = _fill_case(c)
    a = np.asfortranarray(before.copy())
    O.fill_ghost(a, c["bc_x"], c["bc_y"])
    assert np.array_equal(a, after)
