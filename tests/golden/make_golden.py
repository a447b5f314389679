"""Generate the golden fixtures from the REFERENCE itself (run in the build
container, where /root/reference exists; the GPU box never runs this).

    python tests/golden/make_golden.py

Writes tests/golden/reference_golden.json:
  * "steps": first-order runs of reference wavesweep.driver.step on seeded
    inputs (including BASELINE configs[0] = C1 at full size, 256^2 x 100
    steps): every dt / max speed and a SHA-256 of the final state
    (canonicalised with +0.0 so -0/+0 compare like np.array_equal).
  * "kernels": reference rp_* outputs on seeded batches (both directions).
  * "errors": the reference's SweepError text for poisoned cells.
and tests/golden/oracle_golden.json (same format) from the builder's oracle
extension for the solvers/limiters the reference lacks — regression
fixtures only ("parity unpinned").
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def state_hash(q: np.ndarray) -> str:
    c = np.asfortranarray(q, dtype=np.float64) + 0.0
    return hashlib.sha256(c.tobytes(order="F")).hexdigest()


def load_reference():
    src = "/root/reference/pkg/src"
    tmp = tempfile.mkdtemp()
    shutil.copytree(src, os.path.join(tmp, "src"))   # keep caches out of the read-only tree
    sys.path.insert(0, os.path.join(tmp, "src"))
    import wavesweep  # noqa: F401
    import wavesweep.oracles  # noqa: F401
    return wavesweep


STEP_CASES = [
    # name, kernel, params, nx, ny, steps, bc_x, bc_y, seed
    ("c1-full", "acoustics-const", {"rho": 1.0, "bulk": 4.0}, 256, 256, 100,
     "extrapolate", "extrapolate", 0),
    ("acoustics-const-per", "acoustics-const", {"rho": 1.3, "bulk": 2.1}, 37, 29, 6,
     "periodic", "periodic", 1),
    ("acoustics-var-ext", "acoustics-var", {}, 37, 29, 6, "extrapolate", "extrapolate", 2),
    ("acoustics-var-mix", "acoustics-var", {}, 31, 40, 6, "periodic", "extrapolate", 3),
    ("euler-per", "euler", {"gamma": 1.4}, 37, 29, 6, "periodic", "periodic", 4),
    ("euler-ext", "euler", {"gamma": 1.4}, 45, 21, 6, "extrapolate", "extrapolate", 5),
    ("advection-per", "advection", {"u": 0.7, "v": -1.3}, 33, 26, 8, "periodic", "periodic", 6),
    ("advection-ext", "advection", {"u": -0.4, "v": 2.0}, 20, 31, 8, "extrapolate",
     "extrapolate", 7),
]


def case_input(name, kernel, nx, ny, seed):
    from helpers import random_state
    if name == "c1-full":
        from paper_1308_1464_b200 import configs
        c = configs.c1_acoustics()
        return c.q, None, c.dx, c.dy
    q, aux = random_state(kernel, nx, ny, seed)
    return q, aux, 1.0 / nx, 1.3 / ny


def reference_steps(W):
    out = {}
    for name, kernel, params, nx, ny, steps, bcx, bcy, seed in STEP_CASES:
        q, aux, dx, dy = case_input(name, kernel, nx, ny, seed)
        d = W.DESCRIPTORS[kernel]
        spec = W.GridSpec(nx=nx, ny=ny, dx=dx, dy=dy, num_eqn=d.num_eqn, num_aux=d.num_aux)
        st, ax = W.StateField(spec), W.AuxField(spec)
        st.data[...] = q
        if aux is not None:
            ax.data[...] = aux
        cfg = W.SimulationConfig(spec=spec, kernel=kernel, ic=W.DEFAULT_IC[kernel],
                                 num_steps=steps, bc_x=W.BoundaryCondition(bcx),
                                 bc_y=W.BoundaryCondition(bcy), kernel_params=params)
        ctl = W.TimestepController(0.9)
        reps = [W.step(st, ax, cfg, ctl)[1] for _ in range(steps)]
        out[name] = {"kernel": kernel, "params": params, "nx": nx, "ny": ny, "steps": steps,
                     "bc_x": bcx, "bc_y": bcy, "seed": seed, "dx": dx, "dy": dy,
                     "dts": [r.dt for r in reps], "msx": [r.max_speed_x for r in reps],
                     "msy": [r.max_speed_y for r in reps], "cfl": [r.cfl for r in reps],
                     "q_sha256": state_hash(st.data),
                     "q_probe": [float(st.data[c, 2 + nx // 2, 2 + ny // 3])
                                 for c in range(d.num_eqn)]}
        print("ref", name, out[name]["dts"][-1])
    return out


def reference_kernels(W):
    from wavesweep.kernels import (AcousticsParams, Direction, EulerParams, rp_acoustics_const,
                                   rp_acoustics_var, rp_advection, rp_euler)
    from wavesweep.oracles import random_gas_states
    rng = np.random.default_rng(20240817)
    out = {}
    n = 64
    for dname, d in (("x", Direction.X), ("y", Direction.Y)):
        ql, qr = rng.normal(size=(2, 1, n))
        r = rp_advection(d, ql, qr, 1.25, -0.75)
        out[f"advection-{dname}"] = dict(ql=ql.tolist(), qr=qr.tolist(),
                                          params={"u": 1.25, "v": -0.75},
                                          amdq=r.amdq.tolist(), apdq=r.apdq.tolist(),
                                          speeds=r.speeds.tolist(), waves=r.waves.tolist())
        ql, qr = rng.normal(size=(2, 3, n))
        r = rp_acoustics_const(d, ql, qr, AcousticsParams(1.7, 2.9))
        out[f"acoustics-const-{dname}"] = dict(ql=ql.tolist(), qr=qr.tolist(),
                                                params={"rho": 1.7, "bulk": 2.9},
                                                amdq=r.amdq.tolist(), apdq=r.apdq.tolist(),
                                                speeds=r.speeds.tolist(), waves=r.waves.tolist())
        ql, qr = rng.normal(size=(2, 3, n))
        al, ar = rng.uniform(0.2, 5.0, (2, 2, n))
        r = rp_acoustics_var(d, ql, qr, al, ar)
        out[f"acoustics-var-{dname}"] = dict(ql=ql.tolist(), qr=qr.tolist(), auxl=al.tolist(),
                                              auxr=ar.tolist(), params={},
                                              amdq=r.amdq.tolist(), apdq=r.apdq.tolist(),
                                              speeds=r.speeds.tolist(), waves=r.waves.tolist())
        ql = random_gas_states(rng, n, 1.4)
        qr = random_gas_states(rng, n, 1.4)
        r = rp_euler(d, ql, qr, EulerParams(1.4))
        out[f"euler-{dname}"] = dict(ql=ql.tolist(), qr=qr.tolist(), params={"gamma": 1.4},
                                      amdq=r.amdq.tolist(), apdq=r.apdq.tolist(),
                                      speeds=r.speeds.tolist(), waves=r.waves.tolist())
    return out


def reference_errors(W):
    from helpers import random_state
    out = {}
    for kernel, params, comp, val in (("euler", {"gamma": 1.4}, 0, -1.0),
                                      ("euler", {"gamma": 1.4}, 3, 0.0),
                                      ("acoustics-const", {"rho": 1.0, "bulk": 1.0}, 1, np.nan),
                                      ("acoustics-var", {}, 0, np.inf)):
        nx, ny = 12, 9
        q, aux = random_state(kernel, nx, ny, 8)
        q[comp, 2 + 5, 2 + 3] = val
        d = W.DESCRIPTORS[kernel]
        spec = W.GridSpec(nx=nx, ny=ny, dx=1 / nx, dy=1 / ny, num_eqn=d.num_eqn,
                          num_aux=d.num_aux)
        st, ax = W.StateField(spec), W.AuxField(spec)
        st.data[...] = q
        if aux is not None:
            ax.data[...] = aux
        cfg = W.SimulationConfig(spec=spec, kernel=kernel, ic=W.DEFAULT_IC[kernel],
                                 num_steps=1, bc_x=W.BoundaryCondition.EXTRAPOLATE,
                                 bc_y=W.BoundaryCondition.EXTRAPOLATE, kernel_params=params)
        try:
            W.step(st, ax, cfg, W.TimestepController(0.9))
            msg = None
        except W.SweepError as e:
            msg = str(e)
        key = f"{kernel}-c{comp}-{val}"
        out[key] = {"kernel": kernel, "params": params, "comp": comp, "value": repr(val),
                    "nx": nx, "ny": ny, "seed": 8, "message": msg}
        print("err", key, msg)
    return out


ORACLE_CASES = [
    # name, kernel, nx, ny, steps, order, limiter, bc, seed
    ("sw-mc-ext", "shallow-water-roe", 45, 35, 5, 2, "mc", "extrapolate", 1),
    ("sw-superbee-per", "shallow-water-roe", 40, 33, 5, 2, "superbee", "periodic", 2),
    ("hlle-minmod-ext", "euler-hlle", 45, 35, 5, 2, "minmod", "extrapolate", 3),
    ("hlle-mc-per", "euler-hlle", 40, 33, 5, 2, "mc", "periodic", 4),
    ("acvar-mc-ext", "acoustics-var", 45, 35, 5, 2, "mc", "extrapolate", 5),
    ("euler-roe-mc-ext", "euler", 45, 35, 5, 2, "mc", "extrapolate", 6),
]


def oracle_steps():
    from helpers import PARAMS, oracle_run, random_state
    out = {}
    for name, kernel, nx, ny, steps, order, lim, bc, seed in ORACLE_CASES:
        q, aux = random_state(kernel, nx, ny, seed)
        oq, reps = oracle_run(kernel, q, aux, nx, ny, 1 / nx, 1.3 / ny, steps=steps,
                              order=order, limiter=lim, bc_x=bc, bc_y=bc)
        out[name] = {"kernel": kernel, "params": PARAMS[kernel], "nx": nx, "ny": ny,
                     "steps": steps, "order": order, "limiter": lim, "bc_x": bc, "bc_y": bc,
                     "seed": seed, "dx": 1 / nx, "dy": 1.3 / ny,
                     "dts": [r.dt for r in reps], "q_sha256": state_hash(oq)}
    # C2 at a reduced size (the bench workload's recipe, 128^2 x 40 steps)
    from paper_1308_1464_b200 import configs
    c = configs.c2_shallow_water(128, steps=40)
    oq, reps = oracle_run(c.kernel, c.q, None, c.nx, c.ny, c.dx, c.dy, steps=40, order=2,
                          limiter="mc", bc_x="extrapolate", bc_y="extrapolate")
    out["c2-128"] = {"kernel": c.kernel, "params": c.kernel_params, "nx": 128, "ny": 128,
                     "steps": 40, "order": 2, "limiter": "mc", "bc_x": "extrapolate",
                     "bc_y": "extrapolate", "recipe": "configs.c2_shallow_water(128)",
                     "dx": c.dx, "dy": c.dy, "dts": [r.dt for r in reps],
                     "q_sha256": state_hash(oq)}
    return out


def main():
    W = load_reference()
    ref = {"generator": "tests/golden/make_golden.py", "source": "reference wavesweep",
           "steps": reference_steps(W), "kernels": reference_kernels(W),
           "errors": reference_errors(W)}
    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(ref, f)
    orc = {"generator": "tests/golden/make_golden.py", "source": "builder oracle extension",
           "steps": oracle_steps()}
    with open(os.path.join(HERE, "oracle_golden.json"), "w") as f:
        json.dump(orc, f, indent=0)
    print("wrote fixtures")


if __name__ == "__main__":
    main()
