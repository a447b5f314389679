"""Benchmark matrix in the reference's CSV format, for the CUDA step.

Mirrors reference ``wavesweep/bench.py`` (matrix enumeration :150-188,
BenchConfig validation :43-80, record/speedup/efficiency :191-204, CSV
writer :211-234): kernel x size x strategy x backend x threads, median of
repetitions, and a bitwise guard against a twin run.  The backends here are
the two ways a caller drives the GPU:

* ``cuda``      — ``driver.step`` per step: host state uploaded, one device
                  step, report polled, state downloaded (the reference's own
                  per-step API contract, so directly comparable to its rows);
* ``cuda-run``  — device-resident loop: one upload, ``ws_run`` graph replays,
                  one download at the end.

The ``cuda`` row is the twin: a ``cuda-run`` whose final state is not
bitwise identical to it aborts the bench (BenchGuardError, as the
reference's threaded-vs-serial guard :176-183).  ``speedup`` is relative to
the ``cuda`` row; ``threads`` is the GPU count (1: one process drives one
GPU; multi-GPU rows come from ``bench.py --gpus N`` under torchrun).

The CSV is byte-for-byte the reference's eleven-column format, so the
reference's own ``parse_csv`` (bench.py:236-264) reads it back.  The roofline
columns (algorithmic bytes per cell-update = q read + aux read + q written,
achieved GB/s, fraction of the measured HBM peak from MEASURED_PEAKS.json)
go to a sidecar file (``--roofline-out``, :func:`emit_roofline_csv`).

    python -m paper_1308_1464_b200.benchmatrix --kernels shallow-water-roe \
        --sizes 1024x1024 --order 2 --limiter mc --out matrix.csv
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from dataclasses import dataclass

import numpy as np

from .device import Cuda
from .driver import (DEFAULT_IC, LIMITERS, SimulationConfig, TimestepController,
                     initial_condition, session_for, step)
from .kernels import DESCRIPTORS
from .sweep import CellWise, RowWise, Strategy, Tiled

CSV_HEADER = ("kernel,nx,ny,strategy,backend,threads,steps,"
              "ms_per_step,mcells_per_s,speedup,efficiency")
ROOFLINE_KEY = "kernel,nx,ny,strategy,backend"
ROOFLINE_HEADER = "bytes_per_cell,achieved_gbs,hbm_frac"
BACKEND_NAMES = ("cuda", "cuda-run")
EFFICIENCY_FLAG = 1.5
FALLBACK_HBM_GBS = 8000.0   # north_star nominal, when MEASURED_PEAKS.json is absent


class BenchGuardError(RuntimeError):
    """A cuda-run final state differed bitwise from its per-step twin."""


@dataclass(frozen=True)
class BenchConfig:
    kernels: tuple[str, ...]
    sizes: tuple[tuple[int, int], ...]
    strategies: tuple[Strategy, ...] = (Tiled(),)
    backends: tuple[str, ...] = BACKEND_NAMES
    threads: tuple[int, ...] = (1,)
    steps: int = 5
    warmup: int = 2
    repetitions: int = 5
    cfl: float = 0.9
    order: int = 1
    limiter: str = "none"
    precision: str = "f64"
    device: int = 0
    out: str | None = None

    def __post_init__(self):
        for name, values in (("kernels", self.kernels), ("sizes", self.sizes),
                             ("strategies", self.strategies),
                             ("backends", self.backends), ("threads", self.threads)):
            if not values:
                raise ValueError(f"{name} must be nonempty")
        for k in self.kernels:
            if k not in DESCRIPTORS:
                raise ValueError(f"unknown kernel {k!r}")
        for b in self.backends:
            if b not in BACKEND_NAMES:
                raise ValueError(f"unknown backend {b!r}")
        for t in self.threads:
            if t != 1:
                raise ValueError(f"one process drives one GPU; threads must be 1, got {t} "
                                 "(multi-GPU rows: bench.py --gpus N under torchrun)")
        for nx, ny in self.sizes:
            if nx < 1 or ny < 1:
                raise ValueError(f"grid sizes must be >= 1, got {nx}x{ny}")
        if self.steps < 1:
            raise ValueError(f"steps must be >= 1, got {self.steps}")
        if self.warmup < 0:
            raise ValueError(f"warmup must be >= 0, got {self.warmup}")
        if self.repetitions < 1:
            raise ValueError(f"repetitions must be >= 1, got {self.repetitions}")
        if self.order not in (1, 2):
            raise ValueError(f"order must be 1 or 2, got {self.order}")
        if self.limiter not in LIMITERS:
            raise ValueError(f"unknown limiter {self.limiter!r}")


@dataclass
class BenchRecord:
    kernel: str
    nx: int
    ny: int
    strategy: str
    backend: str
    threads: int
    steps: int
    ms_per_step: float
    mcells_per_s: float
    speedup: float
    efficiency: float
    bytes_per_cell: int
    achieved_gbs: float
    hbm_frac: float


def strategy_name(strategy: Strategy) -> str:
    if isinstance(strategy, RowWise):
        return "rowwise"
    if isinstance(strategy, CellWise):
        return "cellwise"
    if isinstance(strategy, Tiled):
        return "tiled"
    raise TypeError(f"unknown strategy {strategy!r}")


def bytes_per_cell(kernel: str, precision: str) -> int:
    d = DESCRIPTORS[kernel]
    return (2 * d.num_eqn + d.num_aux) * (8 if precision == "f64" else 4)


def hbm_peak_gbs() -> float:
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return FALLBACK_HBM_GBS


def _config(kernel, nx, ny, strategy, cfg: BenchConfig, steps) -> SimulationConfig:
    from .grid import GridSpec
    d = DESCRIPTORS[kernel]
    spec = GridSpec(nx=nx, ny=ny, dx=1.0 / nx, dy=1.0 / ny, num_eqn=d.num_eqn,
                    num_aux=d.num_aux)
    return SimulationConfig(spec=spec, kernel=kernel, ic=DEFAULT_IC[kernel],
                            strategy=strategy, backend=Cuda(cfg.device, cfg.precision),
                            num_steps=steps, order=cfg.order, limiter=cfg.limiter)


def _measure_step_api(sim: SimulationConfig, cfg: BenchConfig):
    """Per-step public API (reference _measure_cell, bench.py:126-147)."""
    ctl = TimestepController(cfl_target=cfg.cfl)
    state, aux, _ = initial_condition(sim.ic, sim.spec)
    for _ in range(cfg.warmup):
        step(state, aux, sim, ctl)
    per_rep = []
    for _ in range(cfg.repetitions):
        t0 = time.perf_counter()
        for _ in range(cfg.steps):
            step(state, aux, sim, ctl)
        per_rep.append((time.perf_counter() - t0) * 1e3 / cfg.steps)
    return per_rep, state.interior.copy()


def _measure_device_run(sim: SimulationConfig, cfg: BenchConfig):
    """Device-resident loop: upload once, graph-replayed steps, download once."""
    ctl = TimestepController(cfl_target=cfg.cfl)
    state, aux, _ = initial_condition(sim.ic, sim.spec)
    sess = session_for(sim)
    dt = np.float64 if sess.precision == "f64" else np.float32
    sess.upload(np.asfortranarray(state.data, dtype=dt),
                np.asfortranarray(aux.data, dtype=dt) if sim.spec.num_aux else None)
    native = ctl.native()
    if cfg.warmup:
        sess.run(cfg.warmup, native)
    sess.sync()
    per_rep = []
    for _ in range(cfg.repetitions):
        t0 = time.perf_counter()
        sess.run(cfg.steps, native)
        sess.sync()
        per_rep.append((time.perf_counter() - t0) * 1e3 / cfg.steps)
    res = sess.poll()
    sess.raise_for(res.error)
    state.data[...] = sess.download()
    return per_rep, state.interior.copy()


def _record(kernel, nx, ny, sname, backend, steps, ms, base_ms, bpc, peak) -> BenchRecord:
    total_s = ms * steps / 1e3
    speedup = base_ms / ms
    efficiency = speedup / 1
    if efficiency > EFFICIENCY_FLAG:
        print(f"note: superlinear efficiency {efficiency:.2f} for {kernel} {nx}x{ny} "
              f"{sname} {backend} x1", file=sys.stderr)
    cps = nx * ny * steps / total_s
    gbs = cps * bpc / 1e9
    return BenchRecord(kernel=kernel, nx=nx, ny=ny, strategy=sname, backend=backend,
                       threads=1, steps=steps, ms_per_step=ms, mcells_per_s=cps / 1e6,
                       speedup=speedup, efficiency=efficiency, bytes_per_cell=bpc,
                       achieved_gbs=gbs, hbm_frac=gbs / peak)


def run_bench(cfg: BenchConfig, progress=None) -> list[BenchRecord]:
    """Measure the matrix; records in enumeration order (kernel, size,
    strategy, backend).  The per-step ``cuda`` twin runs for every
    (kernel, size, strategy), requested or not, for speedups and the guard."""
    say = progress or (lambda msg: None)
    peak = hbm_peak_gbs()
    records: list[BenchRecord] = []
    for kernel in cfg.kernels:
        bpc = bytes_per_cell(kernel, cfg.precision)
        for nx, ny in cfg.sizes:
            for strategy in cfg.strategies:
                sname = strategy_name(strategy)
                sim = _config(kernel, nx, ny, strategy, cfg, cfg.steps)
                say(f"{kernel} {nx}x{ny} {sname}: cuda (per-step API twin)")
                base_rep, base_state = _measure_step_api(sim, cfg)
                base_ms = statistics.median(base_rep)
                for backend in cfg.backends:
                    if backend == "cuda":
                        records.append(_record(kernel, nx, ny, sname, "cuda", cfg.steps,
                                               base_ms, base_ms, bpc, peak))
                        continue
                    say(f"{kernel} {nx}x{ny} {sname}: {backend}")
                    rep, state = _measure_device_run(sim, cfg)
                    if not np.array_equal(state, base_state):
                        raise BenchGuardError(
                            f"final state mismatch vs per-step twin: kernel={kernel} "
                            f"size={nx}x{ny} strategy={sname} backend={backend}")
                    records.append(_record(kernel, nx, ny, sname, backend, cfg.steps,
                                           statistics.median(rep), base_ms, bpc, peak))
    return records


def _fmt(x: float) -> str:
    return f"{x:.6g}"


def _open(out):
    if out is None:
        return sys.stdout, False
    if hasattr(out, "write"):
        return out, False
    return open(out, "w", encoding="utf-8"), True


def emit_csv(records: list[BenchRecord], out=None) -> None:
    """Reference emit_csv (bench.py:209-234): the exact eleven-column header
    and rows, 6 significant digits for reals."""
    fh, own = _open(out)
    try:
        fh.write(CSV_HEADER + "\n")
        for r in records:
            fh.write(",".join([
                r.kernel, str(r.nx), str(r.ny), r.strategy, r.backend, str(r.threads),
                str(r.steps), _fmt(r.ms_per_step), _fmt(r.mcells_per_s), _fmt(r.speedup),
                _fmt(r.efficiency)]) + "\n")
    finally:
        if own:
            fh.close()


def emit_roofline_csv(records: list[BenchRecord], out=None) -> None:
    """Sidecar of emit_csv: the row key plus the three roofline columns."""
    fh, own = _open(out)
    try:
        fh.write(ROOFLINE_KEY + "," + ROOFLINE_HEADER + "\n")
        for r in records:
            fh.write(",".join([r.kernel, str(r.nx), str(r.ny), r.strategy, r.backend,
                               str(r.bytes_per_cell), _fmt(r.achieved_gbs),
                               _fmt(r.hbm_frac)]) + "\n")
    finally:
        if own:
            fh.close()


def parse_csv(source) -> list[BenchRecord]:
    """Reference parse_csv (bench.py:236-264): header and eleven fields checked."""
    fh, own = (source, False) if hasattr(source, "read") else (
        open(source, "r", encoding="utf-8"), True)
    try:
        lines = [ln.strip() for ln in fh if ln.strip()]
    finally:
        if own:
            fh.close()
    if not lines or lines[0] != CSV_HEADER:
        raise ValueError("not a bench CSV: bad or missing header")
    out = []
    for ln in lines[1:]:
        p = ln.split(",")
        if len(p) != 11:
            raise ValueError(f"malformed row: {ln!r}")
        out.append(BenchRecord(p[0], int(p[1]), int(p[2]), p[3], p[4], int(p[5]), int(p[6]),
                               float(p[7]), float(p[8]), float(p[9]), float(p[10]),
                               0, 0.0, 0.0))
    return out


def _size(s: str) -> tuple[int, int]:
    a, _, b = s.lower().partition("x")
    return int(a), int(b or a)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1308_1464_b200.benchmatrix")
    ap.add_argument("--kernels", nargs="+", default=["shallow-water-roe"])
    ap.add_argument("--sizes", nargs="+", default=["256x256", "1024x1024"])
    ap.add_argument("--strategies", nargs="+", default=["tiled"],
                    choices=["rowwise", "cellwise", "tiled"])
    ap.add_argument("--backends", nargs="+", default=list(BACKEND_NAMES))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--repetitions", type=int, default=5)
    ap.add_argument("--cfl", type=float, default=0.9)
    ap.add_argument("--order", type=int, default=1)
    ap.add_argument("--limiter", default="none")
    ap.add_argument("--precision", default="f64", choices=["f64", "f32", "f32fast"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--roofline-out", default=None,
                    help="sidecar CSV with bytes/cell, achieved GB/s and the HBM fraction")
    a = ap.parse_args(argv)
    strat = {"rowwise": RowWise(), "cellwise": CellWise(), "tiled": Tiled()}
    cfg = BenchConfig(kernels=tuple(a.kernels), sizes=tuple(_size(s) for s in a.sizes),
                      strategies=tuple(strat[s] for s in a.strategies),
                      backends=tuple(a.backends), steps=a.steps, warmup=a.warmup,
                      repetitions=a.repetitions, cfl=a.cfl, order=a.order,
                      limiter=a.limiter, precision=a.precision, out=a.out)
    recs = run_bench(cfg, progress=lambda m: print(m, file=sys.stderr))
    emit_csv(recs, cfg.out)
    if a.roofline_out:
        emit_roofline_csv(recs, a.roofline_out)
    return 0


if __name__ == "__main__":
    sys.exit(main())
