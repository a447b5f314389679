"""Calibrate the CPU baseline: the reference's own bench harness vs the
numpy oracle port, same machine, same first-order workloads.

Runs in the build container only (imports the reference from a scratch copy
of /root/reference; nothing here travels to the GPU box).  The GPU box's
bench lines time the oracle port (`cpu_baseline.kind = "port"`) because the
reference cannot travel; this file records how the port's speed relates to
the reference's own code path on identical inputs.

    python tools/ref_cpu_calibration.py [--size 512] [--out profiles/r1_cpu_calibration.json]
"""
import argparse
import json
import os
import shutil
import statistics
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def load_reference():
    tmp = tempfile.mkdtemp()
    shutil.copytree("/root/reference/pkg/src", os.path.join(tmp, "src"))
    sys.path.insert(0, os.path.join(tmp, "src"))
    import wavesweep  # noqa: F401
    return wavesweep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_cpu_calibration.json"))
    a = ap.parse_args()
    W = load_reference()
    from wavesweep.bench import BenchConfig, run_bench
    from wavesweep.sweep import Tiled

    from oracle import wavestep_oracle as O
    n = a.size
    threads = os.cpu_count() or 1
    kernels = ("acoustics-const", "acoustics-var", "euler")
    cfg = BenchConfig(kernels=kernels, sizes=((n, n),), strategies=(Tiled(),),
                      backends=("serial", "static", "workstealing"), threads=(threads,),
                      steps=a.steps, warmup=1, repetitions=a.reps)
    recs = run_bench(cfg)
    ref = {}
    for r in recs:
        ref.setdefault(r.kernel, {})[f"{r.backend}x{r.threads}"] = r.mcells_per_s
    port = {}
    for k in kernels:
        d = W.DESCRIPTORS[k]
        spec = W.GridSpec(nx=n, ny=n, dx=1.0 / n, dy=1.0 / n, num_eqn=d.num_eqn,
                          num_aux=d.num_aux)
        st, ax, _ = W.initial_condition(W.DEFAULT_IC[k], spec)
        params = {"acoustics-const": {"rho": 1.0, "bulk": 1.0}, "acoustics-var": {},
                  "euler": {"gamma": 1.4}}[k]
        solver = O.make_solver(k, **params)
        ospec = O.Spec(n, n, 1.0 / n, 1.0 / n)
        q = np.asfortranarray(st.data.copy())
        aux = np.asfortranarray(ax.data.copy()) if d.num_aux else None
        for th in (1, threads):
            ctl = O.Controller(0.9)
            O.step(q, aux, ospec, solver, ctl, bc_x="periodic", bc_y="periodic", order=1,
                   threads=th)
            per = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                for _ in range(a.steps):
                    O.step(q, aux, ospec, solver, ctl, bc_x="periodic", bc_y="periodic",
                           order=1, threads=th)
                per.append((time.perf_counter() - t0) / a.steps)
            port.setdefault(k, {})[f"port x{th}"] = n * n / statistics.median(per) / 1e6
    out = {"machine": f"build container, {threads} cores (os.cpu_count)",
           "workload": f"{n}x{n}, first order, the reference's default IC per kernel, "
                       f"periodic BCs, {a.steps} steps x {a.reps} reps (median)",
           "unit": "Mcell-updates/s",
           "reference_bench_harness": ref, "oracle_port": port,
           "ratio_port_best_over_reference_best": {
               k: max(port[k].values()) / max(ref[k].values()) for k in kernels}}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
