#!/usr/bin/env python
"""Benchmark of the B200 wave-propagation step (contract: see DESIGN.md §7).

Default workload = BASELINE.json configs[4] (C5), the largest single-GPU
configuration: 2D shallow water, Roe + Harten entropy fix, 16384x16384 cells
on the unit square, fp64, MC limiter, second order, CFL 0.9, extrapolation
BCs, h = 1 + 64 seeded Gaussian bumps.  One bench "step" is one time step of
that simulation.  `--config c1..c4` time the other BASELINE configurations.

Metric: cell-updates/s = nx*ny*steps / time (reference bench.py:194-203).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
  python bench.py --impl reference ...      # reference-path CPU arm

N > 1 (torchrun): weak scaling, row strips of nx x ny per rank stacked along
y, halo rows + the CFL max exchanged with NCCL every step (parallel.py);
--strong cuts the 1-GPU grid into N row strips instead (BASELINE C3 / C5
strong-scaling runs: `--config c5 --strong`).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell-updates/sec per step (fp64)"
UNIT = "cell-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--precision", default=None, choices=[None, "f64", "f32", "f32fast"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-ref-code", action="store_true",
                    help="skip timing the reference package's own step (baseline/_ref)")
    ap.add_argument("--device-reduce", action="store_true",
                    help="row-strip path: CFL reduction by the kernels over peer memory "
                         "(symmetric memory) instead of an NCCL all-reduce")
    ap.add_argument("--device-halo", action="store_true",
                    help="row-strip path: halo rows pushed by the update kernel into the "
                         "neighbours' ghost rows over peer memory (implies --device-reduce)")
    ap.add_argument("--strong", action="store_true",
                    help="row-strip path: strong scaling (the 1-GPU grid cut into N strips) "
                         "instead of weak (an N-times taller grid, one 1-GPU strip per rank)")
    ap.add_argument("--eager", action="store_true",
                    help="row-strip path: issue every step from Python instead of replaying "
                         "graphs (ws_run for device collectives, a captured two-step graph "
                         "with the NCCL calls otherwise)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the row-strip (NCCL) path even with one rank (tests it on 1 GPU)")
    ap.add_argument("--size", type=int, default=None,
                    help="override the grid edge (c2/c5 only; size sweeps, not a bench line)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def build_case(name: str, n_ranks: int = 1, precision: str | None = None, device=None,
               size: int | None = None):
    from paper_1308_1464_b200 import configs
    if name == "c5":
        # 16384^2: the 64-bump sum runs in torch on the GPU when one is given
        # (from the numpy 1D factors: the same bits as the host generator)
        c = configs.c5_bumps(size or 16384, dtype=precision or "f64", device=device)
        if c.q is None:
            h = c.meta.pop("h_dev").t().contiguous().cpu().numpy()    # [i][j]
            q = configs._field(3, c.nx, c.ny)
            q[0, 2:2 + c.nx, 2:2 + c.ny] = h
            c.q = q
    elif name == "c2" and size:
        c = configs.c2_shallow_water(size)
    else:
        c = configs.BUILDERS[name]()
    if precision:
        c.dtype = precision
    return c


# the CPU legs time whole steps of a bounded row band of the workload (its
# own grid: the band's cells plus the two rows either side as its ghost
# frame, extrapolation BCs): at most this many cells per sample step
CPU_SAMPLE_CELLS = 1 << 23


def cpu_sample_case(name: str, precision: str | None = None, size: int | None = None):
    """The workload's bounded CPU sample: the whole grid when it has at most
    CPU_SAMPLE_CELLS cells, else the centred row band of that many cells."""
    from paper_1308_1464_b200 import configs
    if name == "c5":
        n = size or 16384
        rows = max(2, min(n, CPU_SAMPLE_CELLS // n))
        j0 = (n - rows) // 2
        c = configs.c5_bumps(n, rows=(j0, j0 + rows))
    else:
        c = build_case(name, size=size)
        if c.cells > CPU_SAMPLE_CELLS:
            rows = max(2, CPU_SAMPLE_CELLS // c.nx)
            j0 = (c.ny - rows) // 2
            sl = slice(j0, j0 + rows + 4)       # band rows + 2 ghost rows each side
            c.q = np.asfortranarray(c.q[:, :, sl])
            if c.aux is not None:
                c.aux = np.asfortranarray(c.aux[:, :, sl])
            c.meta = dict(c.meta, rows=(j0, j0 + rows), ny_full=c.ny)
            c.ny = rows
    if precision:
        c.dtype = precision
    return c


def sample_text(c) -> str:
    j0, j1 = c.meta.get("rows", (0, c.ny))
    if "ny_full" in c.meta and (j0, j1) != (0, c.meta["ny_full"]):
        return (f"rows [{j0}, {j1}) of the {c.nx}x{c.meta['ny_full']} grid as their own "
                f"{c.nx}x{c.ny} grid (same recipe, extrapolation BCs)")
    return f"the whole {c.nx}x{c.ny} grid"


def l2_note(case, ny: int) -> str:
    from paper_1308_1464_b200 import configs
    nb = case.nx * ny * configs.bytes_per_cell(case.kernel, case.dtype) // 2
    if nb > 4 * 126 * 2**20:
        return (f"state {nb / 2**30:.1f} GiB per buffer, larger than the 126 MB L2; "
                "L2 also flushed between timed steps (512 MiB write)")
    return "flushed between timed steps (512 MiB write)"


def workload_config(case, world: int = 1, strong: bool = False, ny_total: int | None = None):
    """The `config` object of the JSON line: identical in both arms."""
    ny = ny_total if ny_total is not None else case.meta.get("ny_full", case.ny)
    wl = case.name
    if world > 1 or strong:
        wl = f"{case.name} in {world} strips (strong)" if strong else \
             f"{case.name} x{world} strips (weak)"
    return {"workload": wl, "kernel": case.kernel, "nx": case.nx, "ny": ny,
            "limiter": case.limiter, "order": case.order, "cfl": case.cfl, "bc": case.bc,
            "precision": case.dtype, "l2": l2_note(case, ny)}


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md "clocks line")

class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# CPU legs (oracle port, numpy + threads; the reference itself is numpy)

def _oracle_setup(case, threads):
    from oracle import wavestep_oracle as O
    solver = O.make_solver(case.kernel, **case.kernel_params)
    spec = O.Spec(case.nx, case.ny, case.dx, case.dy)
    npdt = np.float64 if case.dtype == "f64" else np.float32
    q = np.asfortranarray(case.q, dtype=npdt).copy(order="F")
    aux = np.asfortranarray(case.aux, dtype=npdt).copy(order="F") if case.aux is not None else None
    kw = dict(bc_x=case.bc, bc_y=case.bc, order=case.order, limiter=case.limiter,
              threads=threads)
    return O, solver, spec, q, aux, kw, O.Controller(case.cfl)


def cpu_rate(case, seconds: float, threads: int, max_steps: int = 10**9):
    """Time the oracle port on a bounded sample: whole steps of the sample
    case until `seconds` of CPU work; returns (cell-updates/s, steps, s)."""
    O, solver, spec, q, aux, kw, ctl = _oracle_setup(case, threads)
    O.step(q, aux, spec, solver, ctl, **kw)      # warm-up step (pool start, caches)
    n, t0 = 0, time.perf_counter()
    while n < max_steps:
        O.step(q, aux, spec, solver, ctl, **kw)
        n += 1
        if time.perf_counter() - t0 >= seconds:
            break
    el = time.perf_counter() - t0
    return case.nx * case.ny * n / el, n, el


# the reference package itself, installed by bench setup into baseline/_ref
# (pip install --target baseline/_ref /root/reference; it travels with the
# repo to the GPU box).  It has no shallow-water solver, no limiter and no
# second order, so its own code path is timed on its closest kernel.
REF_CLOSEST = {"shallow-water-roe": "euler", "euler-hlle": "euler", "euler": "euler",
               "acoustics-const": "acoustics-const", "acoustics-var": "acoustics-var",
               "advection": "advection"}


def reference_code_path(sample, budget_s: float = 20.0):
    """Time the reference's own ``wavesweep.driver.step`` (first order) on the
    sample band with its three backends through ``for_each_unit`` (reference
    bench.py:126-147 method: warm-up step, repetitions, median ms/step)."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "wavesweep")):
        return {"unavailable": "reference package not installed in baseline/_ref"}
    if path not in sys.path:
        sys.path.insert(0, path)
    import wavesweep
    from wavesweep import driver as RD
    from wavesweep.grid import BoundaryCondition, GridSpec, StateField, AuxField
    from wavesweep.parallel import Serial, StaticThreads, WorkStealing
    from wavesweep.sweep import CellWise
    kern = REF_CLOSEST[sample.kernel]
    ncores = os.cpu_count() or 1
    g = 2
    neq = {"euler": 4, "acoustics-const": 3, "acoustics-var": 3, "advection": 1}[kern]
    naux = 2 if kern == "acoustics-var" else 0
    # the reference grid needs dx, dy only for dt; the sample's own widths
    spec = GridSpec(nx=sample.nx, ny=sample.ny, dx=sample.dx, dy=sample.dy, num_eqn=neq,
                    num_aux=naux)
    st = StateField(spec)
    q = sample.q
    if kern == "euler" and sample.kernel == "shallow-water-roe":
        # gas at rest with rho = p = h: an admissible Euler state from the band
        h = q[0]
        st.data[0] = h
        st.data[3] = h / 0.4
        params = {"gamma": 1.4}
    else:
        st.data[...] = q[:neq]
        params = dict(sample.kernel_params)
        if sample.kernel == "euler-hlle":
            params = {"gamma": params.get("gamma", 1.4)}
    aux = None
    if naux:
        aux = AuxField(spec)
        aux.data[...] = sample.aux
    ext = BoundaryCondition.EXTRAPOLATE
    ctl = RD.TimestepController(cfl_target=min(sample.cfl, 0.9))
    out = {"package": f"wavesweep {getattr(wavesweep, '__version__', '')}".strip(),
           "kernel": kern, "order": 1, "strategy": "cellwise", "cores": ncores,
           "sample": f"{sample_text(sample)}; "
                     + ("Euler gas at rest with rho = p = h (closest reference kernel: "
                        "it has no shallow-water solver)" if kern != sample.kernel
                        else "the sample's own state"),
           "backends": {}}
    per = budget_s / 3.0
    for name, be in (("serial", Serial()), ("static", StaticThreads(ncores)),
                     ("workstealing", WorkStealing(ncores))):
        cfg = RD.SimulationConfig(spec=spec, kernel=kern, ic=RD.DEFAULT_IC[kern],
                                  strategy=CellWise(), backend=be, bc_x=ext, bc_y=ext,
                                  num_steps=1, kernel_params=params)
        s_ = st.copy()
        a_ = aux.copy() if aux is not None else None
        t0 = time.perf_counter()
        RD.step(s_, a_, cfg, ctl)          # warm-up (thread pool start)
        first = time.perf_counter() - t0
        ms = []
        while len(ms) < 3 and (sum(ms) / 1e3 + first) < per:
            t0 = time.perf_counter()
            RD.step(s_, a_, cfg, ctl)
            ms.append((time.perf_counter() - t0) * 1e3)
        if not ms:
            ms = [first * 1e3]
        med = statistics.median(ms)
        out["backends"][name] = {"ms_per_step": med, "reps": len(ms),
                                 "value": sample.nx * sample.ny / (med / 1e3)}
    best = max(out["backends"], key=lambda k: out["backends"][k]["value"])
    out["best"] = best
    out["value"] = out["backends"][best]["value"]
    out["unit"] = UNIT
    return out


def reference_arm(args):
    """`--impl reference`: the reference path's CPU implementation on the
    host cores -- the oracle port of the full second-order step (the
    reference package has neither the solvers nor the limiters of the
    workload) on the bounded sample, exactly --warmup + --steps time steps;
    the reference package's own first-order step is timed beside it."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    sample = cpu_sample_case(args.config, precision=args.precision, size=args.size)
    threads = os.cpu_count() or 1
    O, solver, spec, q, aux, kw, ctl = _oracle_setup(sample, threads)
    for _ in range(args.warmup):
        O.step(q, aux, spec, solver, ctl, **kw)
    k = args.steps
    t0 = time.perf_counter()
    for _ in range(k):
        O.step(q, aux, spec, solver, ctl, **kw)
    el = time.perf_counter() - t0
    v = sample.nx * sample.ny * k / el
    ref_code = None
    if not args.no_ref_code:
        try:
            ref_code = reference_code_path(sample)
        except Exception as e:  # reported, never fatal for the arm
            ref_code = {"unavailable": f"{type(e).__name__}: {e}"}
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": k, "warmup": args.warmup, "ms_per_step": el * 1e3 / k,
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None, "dtype": sample.dtype, "data": "synthetic",
        "config": workload_config(sample, world, args.strong,
                                  ny_total=sample_ny_total(sample, world, args.strong)),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{k} time steps (after {args.warmup} warm-up) of "
                                   f"{sample_text(sample)}, numpy oracle port of the "
                                   f"second-order step with {threads} threads",
                         "reference_code_path": ref_code},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def sample_ny_total(sample, world, strong):
    ny = sample.meta.get("ny_full", sample.ny)
    return ny if (strong or world == 1) else ny * world


def cpu_baseline_block(case_name, args, precision=None, size=None):
    """cpu_baseline of the GPU arm's line (rank 0, N = 1)."""
    sample = cpu_sample_case(case_name, precision=precision, size=size)
    threads = os.cpu_count() or 1
    v, n, el = cpu_rate(sample, args.cpu_seconds, threads)
    out = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"{n} time steps of {sample_text(sample)} in {el:.1f} s, numpy oracle "
                     f"port of the second-order step with {threads} threads"}
    if not args.no_ref_code:
        try:
            out["reference_code_path"] = reference_code_path(sample)
        except Exception as e:
            out["reference_code_path"] = {"unavailable": f"{type(e).__name__}: {e}"}
    return out


# ---------------------------------------------------------------------------
# GPU arm

def gpu_arm(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.force_sharded:
        return gpu_arm_sharded(args, rank, world, local)

    from paper_1308_1464_b200 import DeviceGrid, _abi, make_kernel, configs
    case = build_case(args.config, precision=args.precision, device=dev, size=args.size)
    prec = case.dtype
    kernel = make_kernel(case.kernel, **case.kernel_params)
    g = DeviceGrid(case.nx, case.ny, case.dx, case.dy, kernel, order=case.order,
                   limiter=case.limiter, bc_x=case.bc, bc_y=case.bc, precision=prec,
                   device=local)
    npdt = np.float64 if prec == "f64" else np.float32
    host_q = np.asfortranarray(case.q, dtype=npdt)
    host_aux = np.asfortranarray(case.aux, dtype=npdt) if case.aux is not None else None
    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream
    ctl = _abi.make_ctl(case.cfl)
    cells = case.nx * case.ny
    bpc = configs.bytes_per_cell(case.kernel, prec)
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device=dev)

    g.upload(host_q, host_aux, stream=sp)
    for _ in range(args.warmup):
        g.step(ctl, stream=sp)
    res = g.poll()
    g.raise_for(res.error)

    dyn = not (case.kernel.startswith("acoustics"))
    k = args.steps

    def timed_loop(split, g=g):
        # events bracket each step (split: also between the two kernels, which
        # costs the programmatic overlap of the pre-pass tail with the update's
        # launch, so the headline uses the unsplit loop)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(k)]
        with torch.cuda.stream(stream):
            # keep the GPU busy while the host enqueues the whole timed loop, so
            # event gaps are device time, not Python/ctypes launch latency
            torch.cuda._sleep(int(2e6 + 4e5 * k))
            for i in range(k):
                flush.zero_()                     # L2 flush between timed steps
                ev[i][0].record(stream)
                if dyn:
                    g.phase_speeds(stream=sp)
                    if split:
                        ev[i][1].record(stream)
                    g.phase_update(ctl, stream=sp)
                else:
                    g.step(ctl, stream=sp)
                    if split:
                        ev[i][1].record(stream)
                ev[i][2].record(stream)
        torch.cuda.synchronize()
        return ev

    l0 = g.launches()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        ev = timed_loop(split=False)
    launches = g.launches() - l0
    res = g.poll()
    g.raise_for(res.error)
    total_ms = sum(ev[i][0].elapsed_time(ev[i][2]) for i in range(k))
    ms_per_step = total_ms / k
    value = cells * k / (total_ms / 1e3)
    # per-kernel split (second loop, same steps): pre-pass | update
    ev = timed_loop(split=True)
    res = g.poll()
    g.raise_for(res.error)
    if dyn:
        t_spd = [ev[i][0].elapsed_time(ev[i][1]) for i in range(k)]
        t_upd = [ev[i][1].elapsed_time(ev[i][2]) for i in range(k)]
    else:
        t_spd = [0.0] * k
        t_upd = [ev[i][0].elapsed_time(ev[i][1]) for i in range(k)]

    # dominant kernel: the fused update; algorithmic bytes = q read + aux read + q write
    upd_ms = statistics.mean(t_upd)
    peak, peak_kind = measured_peak_hbm()
    achieved = cells * bpc / (upd_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "kernel": "k_update",
                "peak_kind": peak_kind, "kernel_ms": upd_ms,
                "speeds_kernel_ms": statistics.mean(t_spd) if dyn else 0.0,
                "algorithmic_bytes_per_cell": bpc,
                "timing": "CUDA events on the launching stream around each kernel, in a second "
                          "loop of the same K steps (an event between the two kernels costs the "
                          "programmatic overlap, so the headline loop has none)"}
    roofline["kernel"] = "k_update_w"
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                # entries per config, and per config + precision for fp32
                pr = json.load(f).get(args.config if prec == "f64" else f"{args.config}_{prec}", {})
            roofline["traffic"] = pr.get("bytes_per_launch")
            if pr.get("fp64_instr_per_cell_approx"):
                # the binding resource: FP64 pipe, from the ncu capture
                ipc = pr.get("fp64_instr_per_cell_approx")
                pk = pr.get("fp64_peak_instr_per_s")
                ach = ipc * cells / (upd_ms / 1e3) if ipc else None
                roofline["fp64"] = {"pipe_active_frac_ncu": pr["fp64_pipe_active_pct"] / 100.0,
                                    "instr_per_cell": ipc,
                                    "achieved_instr_per_s": ach,
                                    "peak_instr_per_s": pk,
                                    "frac": (ach / pk) if (ach and pk) else None,
                                    "note": "FP64 warp-lane instructions per cell from the ncu "
                                            "capture x cells / event-timed update kernel, "
                                            "against the measured DFMA peak",
                                    "peak_source": pr.get("fp64_peak_source")}
            if pr.get("instr_per_cell"):
                # the first binding resource: issue (one warp instruction per
                # clock and scheduler)
                ic = pr["instr_per_cell"] * cells / (upd_ms / 1e3)
                roofline["issue"] = {"instr_per_cell": pr["instr_per_cell"],
                                     "achieved_instr_per_s": ic,
                                     "peak_instr_per_s": pr["issue_peak_instr_per_s"],
                                     "frac": ic / pr["issue_peak_instr_per_s"],
                                     "issue_active_frac_ncu": pr["issue_active_pct"] / 100.0,
                                     "note": "warp-lane instructions per cell from the ncu "
                                             "capture x cells / event-timed update kernel, "
                                             "against 148 SMs x 4 schedulers x 32 lanes x "
                                             "1965 MHz"}
        except Exception:
            pass

    # whole simulation, device resident: the configured number of steps via graphs
    # (one untimed run first so graph capture/instantiation is not timed)
    g.upload(host_q, host_aux, stream=sp)
    g.run(min(case.steps, 8), ctl, stream=sp)
    torch.cuda.synchronize()
    g.poll()
    g.upload(host_q, host_aux, stream=sp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g.run(case.steps, ctl, stream=sp)
    e1.record(stream)
    torch.cuda.synchronize()
    res_run = g.poll()
    g.raise_for(res_run.error)
    sim_ms = e0.elapsed_time(e1)

    # The default CFL pre-pass of shallow water and Euler probes only the tiles
    # that can hold the step's maximum.  Twin handle with
    # WS_SPEEDS=exact (every edge probed): its timing next to ours, and a
    # bitwise guard -- same upload, same steps, states and every report equal.
    exact = None
    if dyn and case.kernel in ("shallow-water-roe", "euler", "euler-hlle"):
        old_env = os.environ.get("WS_SPEEDS")
        os.environ["WS_SPEEDS"] = "exact"
        try:
            g2 = DeviceGrid(case.nx, case.ny, case.dx, case.dy, kernel, order=case.order,
                            limiter=case.limiter, bc_x=case.bc, bc_y=case.bc, precision=prec,
                            device=local)
        finally:
            if old_env is None:
                os.environ.pop("WS_SPEEDS", None)
            else:
                os.environ["WS_SPEEDS"] = old_env
        ns = min(case.steps, 20)
        outs = []
        for h in (g, g2):
            h.upload(host_q, host_aux, stream=sp)
            h.run(ns, ctl, stream=sp)
            torch.cuda.synchronize()
            r = h.poll()
            h.raise_for(r.error)
            outs.append((h.download(), r.reports))
        same = bool(np.array_equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1])
        g2.upload(host_q, host_aux, stream=sp)
        for _ in range(args.warmup):
            g2.step(ctl, stream=sp)
        torch.cuda.synchronize()
        ev2 = timed_loop(split=False, g=g2)
        r2 = g2.poll()
        g2.raise_for(r2.error)
        ms2 = sum(ev2[i][0].elapsed_time(ev2[i][2]) for i in range(k)) / k
        exact = {"value": cells / (ms2 / 1e3), "unit": UNIT, "ms_per_step": ms2,
                 "bitwise_equal_to_default": same, "guard_steps": ns,
                 "note": "same step with the CFL pre-pass probing every edge "
                         "(WS_SPEEDS=exact); the default's tile filter is exact, the guard "
                         "compares the state and every report after guard_steps steps"}
        g2.close()
        if not same:
            raise SystemExit("tile-filtered pre-pass differs from the exact pre-pass")

    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(g, case, host_q, host_aux, ctl, stream, k)
    cpu = None
    if not args.no_cpu:
        # free the host copies of the 6 GB state before the CPU sample runs
        del host_q, host_aux
        case.q = case.aux = None
        cpu = cpu_baseline_block(args.config, args, precision=args.precision, size=args.size)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": k,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": prec, "data": "synthetic",
        "config": workload_config(case),
        "measurement": {"parallelism": "single-gpu",
                        "timed_step": "one time step = CFL pre-pass + fused update",
                        "scaling_note": "N = 1 is the first point of the weak-scaling curve "
                                        "(bench.py --gpus N keeps the per-GPU grid)"},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "exact_prepass": exact,
        "clocks": clk.summary(),
        "simulation": {"steps": case.steps, "ms": sim_ms,
                       "cell_updates_per_s": cells * res_run.steps_done / (sim_ms / 1e3),
                       "l2": "not flushed (whole run, graph replay)"},
    }
    print(json.dumps(line), flush=True)
    g.close()
    return 0


def e2e_leg(g, case, host_q, host_aux, ctl, stream, k):
    """Through the public API with host buffers: per step, pinned H2D of the
    state, one step, D2H of the resulting state (driver.step's contract)."""
    import torch
    sp = stream.cuda_stream
    pin_q = torch.empty(host_q.size, dtype=torch.float64 if host_q.dtype == np.float64
                        else torch.float32, pin_memory=True).numpy()
    pin_q = pin_q.reshape(host_q.shape, order="F")
    pin_q[...] = host_q
    pin_out = torch.empty_like(torch.from_numpy(np.ascontiguousarray(pin_q.ravel(order="F"))),
                               pin_memory=True).numpy().reshape(host_q.shape, order="F")
    pin_aux = None
    if host_aux is not None:
        pin_aux = torch.empty(host_aux.size, dtype=torch.from_numpy(host_aux.ravel()).dtype,
                              pin_memory=True).numpy().reshape(host_aux.shape, order="F")
        pin_aux[...] = host_aux
    n = max(3, min(k, 20))
    for _ in range(2):
        g.upload(pin_q, pin_aux, stream=sp)
        g.step(ctl, stream=sp)
        g.download(pin_out, stream=sp)
    torch.cuda.synchronize()
    # serial: each call returns before the next is issued (download syncs)
    t0 = time.perf_counter()
    for _ in range(n):
        g.upload(pin_q, pin_aux, stream=sp)
        g.step(ctl, stream=sp)
        g.download(pin_out, stream=sp)
    torch.cuda.synchronize()
    el_serial = time.perf_counter() - t0
    res = g.poll()
    g.raise_for(res.error)
    # pipelined: uploads on a second stream, downloads enqueue-only, so the
    # host-to-device copy of step n+1 overlaps the device-to-host copy of
    # step n (PCIe is full duplex); the handle keeps its own operations in
    # issue order across the two streams (include/wavestep.h)
    s_up = torch.cuda.Stream(device=stream.device)
    s_dn = torch.cuda.Stream(device=stream.device)
    up, dn = s_up.cuda_stream, s_dn.cuda_stream
    for _ in range(2):
        g.upload(pin_q, pin_aux, stream=up)
        g.step(ctl, stream=sp)
        g.download(pin_out, stream=dn, wait=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        g.upload(pin_q, pin_aux, stream=up)
        g.step(ctl, stream=sp)
        g.download(pin_out, stream=dn, wait=False)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    res = g.poll()
    g.raise_for(res.error)
    hb = pin_q.nbytes + (pin_aux.nbytes if pin_aux is not None else 0)
    # whole-run variant: one upload, the configured steps, one download
    t1 = time.perf_counter()
    g.upload(pin_q, pin_aux, stream=sp)
    g.run(case.steps, ctl, stream=sp)
    g.download(pin_out, stream=sp)
    el2 = time.perf_counter() - t1
    cells = case.nx * case.ny
    return {"value": cells * n / el, "unit": UNIT, "h2d_bytes_per_step": hb,
            "d2h_bytes_per_step": pin_out.nbytes,
            "api": "per step DeviceGrid.upload (pinned, stream U) / step (stream S) / "
                   "download(wait=False) (pinned, stream D): C ABI ws_upload / ws_step / "
                   "ws_download_async; the H2D of step n+1 and the step overlap the D2H of "
                   "step n",
            "serial_value": cells * n / el_serial,
            "serial_api": "same calls on one stream with the synchronous ws_download",
            "run_value": cells * case.steps / el2,
            "run_api": f"upload once, ws_run({case.steps}) graph replay, download once"}


def gpu_arm_sharded(args, rank, world, local):
    from paper_1308_1464_b200 import parallel
    return parallel.bench_sharded(args, rank, world, local, build_case, Clocks, cpu_rate,
                                  measured_peak_hbm, METRIC, UNIT,
                                  workload_config=workload_config,
                                  cpu_baseline=cpu_baseline_block)


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    return gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
