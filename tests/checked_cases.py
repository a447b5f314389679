"""Parity cases run against the CHECKED build (-DWS_CHECKED=1; the device
analogue of the reference's WAVESWEEP_CHECKED mode, sweep.py:32-33, 78-96).

    WAVESTEP_LIB=paper_1308_1464_b200/_lib/checked/libwavestep.so \\
        python tests/checked_cases.py

Every case must (1) match the oracle bit for bit although every location no
kernel may read holds NaN, (2) report no failed device index check, and (3)
have written every interior cell exactly once per step.  Prints one JSON
line per case; exit status 0 iff all pass.  Driven by test_gpu_checked.py.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

from helpers import PARAMS, device_grid, oracle_run, random_state  # noqa: E402


def single(name, nx, ny, bc, order, limiter, steps, seed, use_run):
    from paper_1308_1464_b200 import _abi
    dx, dy = 1.0 / nx, 1.3 / ny
    q, aux = random_state(name, nx, ny, seed)
    oq, oreps = oracle_run(name, q, aux, nx, ny, dx, dy, steps=steps, order=order,
                           limiter=limiter, bc_x=bc[0], bc_y=bc[1])
    g = device_grid(name, nx, ny, dx, dy, order=order, limiter=limiter, bc_x=bc[0], bc_y=bc[1])
    try:
        g.upload(q, aux)
        c = _abi.make_ctl(0.9)
        if use_run:
            g.run(steps, c)
        else:
            for _ in range(steps):
                g.step(c)
        res = g.poll()
        out = g.download()
        flags, wmin, wmax = g.checked_counts()
    finally:
        g.close()
    ok = (res.error.code == 0 and res.steps_done == steps and np.array_equal(out, oq) and
          [r[0] for r in res.reports] == [r.dt for r in oreps] and flags == 0 and
          wmin == wmax == steps)
    return {"case": f"{name} {nx}x{ny} {bc} o{order} {limiter}", "ok": bool(ok),
            "flags": flags, "writes": [wmin, wmax], "steps": steps}


def single_fast(name, nx, ny, bc, steps, seed):
    """The fp32 throughput mode (f32fast): no index violation, one write per
    cell and step, and the stated bound (rel <= 1e-5) against fp64."""
    from paper_1308_1464_b200 import DeviceGrid, _abi, make_kernel
    dx, dy = 1.0 / nx, 1.3 / ny
    q, aux = random_state(name, nx, ny, seed)
    oq, oreps = oracle_run(name, q, aux, nx, ny, dx, dy, steps=steps, order=2, limiter="mc",
                           bc_x=bc, bc_y=bc)
    g = DeviceGrid(nx, ny, dx, dy, make_kernel(name, **PARAMS[name]), order=2, limiter="mc",
                   bc_x=bc, bc_y=bc, precision="f32fast")
    try:
        g.upload(np.asfortranarray(q, dtype=np.float32),
                 np.asfortranarray(aux, dtype=np.float32) if aux is not None else None)
        g.run(steps, _abi.make_ctl(0.9))
        res = g.poll()
        out = g.download().astype(np.float64)
        flags, wmin, wmax = g.checked_counts()
    finally:
        g.close()
    a, b = out[:, 2:-2, 2:-2], oq[:, 2:-2, 2:-2]
    rel = max(float(np.abs(a[c] - b[c]).max() / max(np.abs(b[c]).max(), 1e-300))
              for c in range(b.shape[0]))
    dts = np.array([r[0] for r in res.reports])
    drel = float(np.abs(dts / np.array([r.dt for r in oreps]) - 1).max())
    ok = (res.error.code == 0 and res.steps_done == steps and rel <= 1e-5 and drel <= 1e-5 and
          flags == 0 and wmin == wmax == steps)
    return {"case": f"f32fast {name} {nx}x{ny} {bc}", "ok": bool(ok), "flags": flags,
            "writes": [wmin, wmax], "rel": rel, "dt_rel": drel}


def canaries_present():
    """The check has teeth: after an upload the padding columns and the
    physical-boundary ghost rows of the device state hold NaN."""
    from cuda.bindings import runtime as rt
    name, nx, ny = "shallow-water-roe", 37, 29
    q, _ = random_state(name, nx, ny, 5)
    g = device_grid(name, nx, ny, 1.0 / nx, 1.0 / ny, order=2, limiter="mc")
    try:
        g.upload(q)
        g.sync()
        ptr, pitch, row = g.state_ptr()
        host = np.empty((ny + 4) * row, dtype=np.float64)
        (rc,) = rt.cudaMemcpy(host.ctypes.data, ptr, host.nbytes,
                              rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        a = host.reshape(ny + 4, 3, pitch)
        ok = (int(rc) == 0 and np.isnan(a[:, :, nx:]).all() and np.isnan(a[:2]).all() and
              np.isnan(a[-2:]).all() and not np.isnan(a[2:-2, :, :nx]).any())
    finally:
        g.close()
    return {"case": "canaries present (padding columns, BC ghost rows = NaN)", "ok": bool(ok)}


def sharded(name, P, bc, dred, dhalo, split=False):
    from test_gpu_multishard import fake_sharded
    nx, ny, steps = 70, 61, 3
    dx, dy = 1.0 / nx, 1.0 / ny
    q, aux = random_state(name, nx, ny, 7)
    oq, oreps = oracle_run(name, q, aux, nx, ny, dx, dy, steps=steps, order=2, limiter="mc",
                           bc_x=bc, bc_y=bc)
    seen = []
    out, reps, errs, strips = fake_sharded(name, q, aux, nx, ny, dx, dy, P, steps, 2, "mc", bc,
                                           device_reduce=dred, device_halo=dhalo,
                                           inspect=lambda g: seen.append(g.checked_counts()),
                                           split_update=split)
    full = np.concatenate(out, axis=2)
    ok = (np.array_equal(full, oq[:, 2:-2, 2:-2]) and all(e.code == 0 for e in errs) and
          all(r == [x.dt for x in oreps] for r in reps) and
          all(f == 0 and lo == hi == steps for f, lo, hi in seen))
    return {"case": f"{name} {P} shards {bc} reduce={dred} halo={dhalo} split={split}",
            "ok": bool(ok),
            "shards": seen}


def main():
    results = [canaries_present()]
    solvers = ["advection", "acoustics-const", "acoustics-var", "euler", "euler-hlle",
               "shallow-water-roe"]
    bcs = [("extrapolate", "extrapolate"), ("periodic", "periodic"), ("periodic", "extrapolate")]
    for name in solvers:
        for bc in bcs:
            results.append(single(name, 37, 29, bc, 2, "mc", 3, 1, False))
        results.append(single(name, 131, 75, ("extrapolate", "extrapolate"), 2, "minmod", 5, 2, True))
        results.append(single(name, 37, 29, ("periodic", "periodic"), 1, "none", 3, 3, False))
    for nx, ny in ((1, 1), (2, 3), (5, 1), (33, 17), (610, 97)):
        results.append(single("shallow-water-roe", nx, ny, ("extrapolate", "extrapolate"), 2,
                              "mc", 3, 4, False))
    # k_run_small (ws_run >= 4 steps on a static-speed grid): 81 tiles, one launch
    results.append(single("acoustics-const", 256, 256, ("extrapolate", "extrapolate"), 2, "mc",
                          12, 5, True))
    results.append(single("acoustics-var", 100, 90, ("periodic", "periodic"), 2, "superbee",
                          7, 6, True))
    for name, bc in (("shallow-water-roe", "extrapolate"), ("euler-hlle", "periodic"),
                     ("acoustics-var", "extrapolate")):
        results.append(single_fast(name, 131, 75, bc, 6, 8))
    for name, P, bc, dred, dhalo in (("shallow-water-roe", 2, "extrapolate", False, False),
                                     ("shallow-water-roe", 3, "periodic", True, False),
                                     ("euler-hlle", 3, "extrapolate", True, True),
                                     ("acoustics-var", 2, "periodic", True, True)):
        results.append(sharded(name, P, bc, dred, dhalo))
    for name, P, bc in (("shallow-water-roe", 3, "periodic"), ("euler-hlle", 2, "extrapolate"),
                        ("acoustics-var", 4, "periodic")):
        results.append(sharded(name, P, bc, False, False, split=True))
    for r in results:
        print(json.dumps(r))
    return 0 if all(r["ok"] for r in results) else 1


if __name__ == "__main__":
    sys.exit(main())
