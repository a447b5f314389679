"""Row-strip decomposition on CPU: world_size 2-3 over gloo (no GPU).

The product orchestration (parallel.exchange_halos / sharded_step /
decode_slot) runs unchanged; only the shard executor is a numpy test double
built from the oracle.  The N-rank result must be bitwise identical to the
single-domain oracle run — the reference's serial-twin guard
(bench.py:181-185) turned into a 1-vs-N guard — including dt, and an
inadmissible cell must be reported identically by every rank.
"""

import os
import pickle
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import PARAMS, random_state
from oracle import wavestep_oracle as O
from paper_1308_1464_b200 import parallel as PL


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class NumpyShard:
    """Oracle-backed shard with the CudaShard interface (test double)."""

    def __init__(self, gq, gaux, strips, rank, name, nx, dx, dy, order, limiter, bc):
        self.j0, self.j1 = strips.bounds(rank)
        self.ny = self.j1 - self.j0
        self.lo, self.hi = strips.neighbours(rank, bc == "periodic")
        self.q = PL.shard_block(gq, self.j0, self.j1).copy(order="F")
        self.aux = PL.shard_block(gaux, self.j0, self.j1).copy(order="F") if gaux is not None else None
        self.spec = O.Spec(nx, self.ny, dx, dy)
        self.solver = O.make_solver(name, **PARAMS[name])
        self.nx, self.order, self.limiter, self.bc = nx, order, limiter, bc
        self.reports, self.error = [], None
        self.halos_primed = False       # the first step exchanges the current rows
        self.calls = []

    def halo_views(self, which="current"):
        # the double updates in place: after phase_update_boundary the next
        # state is self.q itself
        self.calls.append(f"halo_views:{which}")
        n = self.ny
        self._recv = (torch.zeros(self.q[:, :, 0:2].shape, dtype=torch.float64),
                      torch.zeros(self.q[:, :, 0:2].shape, dtype=torch.float64))
        return (torch.from_numpy(np.ascontiguousarray(self.q[:, :, 2:4])),
                torch.from_numpy(np.ascontiguousarray(self.q[:, :, n:n + 2])),
                self._recv[0], self._recv[1])

    def halo_received(self):
        self.calls.append("halo_wait")
        n = self.ny
        if self.lo is not None:
            self.q[:, :, 0:2] = self._recv[0].numpy()
        if self.hi is not None:
            self.q[:, :, n + 2:n + 4] = self._recv[1].numpy()

    def _fill(self, a):
        if a is None or a.shape[0] == 0:
            return
        O._fill(a, self.nx, 2, self.bc, 1)          # x pass over every row
        n = self.ny
        if self.lo is None:                          # physical bottom (extrapolate)
            a[:, :, 0:2] = a[:, :, 2:3]
        if self.hi is None:
            a[:, :, n + 2:n + 4] = a[:, :, n + 1:n + 2]

    def phase_speeds(self):
        if self.lo is None and self.hi is None and self.bc == "periodic":
            O.fill_ghost(self.q, "periodic", "periodic")
            if self.aux is not None:
                O.fill_ghost(self.aux, "periodic", "periodic")
        else:
            self._fill(self.q)
            self._fill(self.aux)
        self.res = O._solve_band(self.q, self.aux, self.spec, self.solver, 0, self.ny,
                                 self.order)
        key = 0
        if self.res.cands:
            best = min(self.res.cands, key=lambda c: c[0])
            d, _, stage, comp, i, jl = best[0]
            jg = self.j0 + jl
            width = self.nx + 1 if d == 0 else self.nx
            chunk = jg // max(1, 32768 // width)
            k = (d << 62) | (chunk << 44) | (stage << 40) | (comp << 37) | (i << 18) | jg
            key = PL.NKEY_MAX - k
        bits = np.array([self.res.max_x, self.res.max_y]).view(np.int64)
        self._slot = torch.tensor([int(bits[0]), int(bits[1]), key], dtype=torch.int64)

    def phase_speeds_interior(self):
        # the double computes everything after the halos landed
        pass

    def phase_speeds_boundary(self):
        self.phase_speeds()

    def slot_view(self):
        return self._slot

    def slot_reduced(self):
        self.msx, self.msy, self.key = PL.decode_slot(self._slot.tolist())

    def phase_update_boundary(self, ctl):
        self.calls.append("update:boundary")
        self.phase_update(ctl)           # the double updates everything here

    def phase_update_interior(self, ctl):
        self.calls.append("update:interior")

    def phase_update(self, ctl):
        if self.error is not None:
            return
        if self.key is not None:
            self.error = self.key
            return
        dt = O.choose_dt(self.msx, self.msy, self.spec.dx, self.spec.dy, O.Controller(ctl))
        O._update_band(self.q, self.spec, self.res, dt, self.order, self.limiter)
        self.reports.append((dt, self.msx, self.msy))


def _worker(rank, world, port, args, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    name, gq, gaux, nx, ny, dx, dy, order, limiter, bc, steps = args
    strips = PL.RowStrips(ny, world)
    sh = NumpyShard(gq, gaux, strips, rank, name, nx, dx, dy, order, limiter, bc)
    for _ in range(steps):
        PL.sharded_step(dist, sh, strips, rank, bc == "periodic", 0.9)
        if sh.error is not None:
            break
    with open(os.path.join(outdir, f"r{rank}.pkl"), "wb") as f:
        pickle.dump({"j0": sh.j0, "j1": sh.j1, "q": sh.q[:, 2:-2, 2:-2], "reports": sh.reports,
                     "error": sh.error}, f)
    dist.destroy_process_group()


def run_sharded(world, *args):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, free_port(), args, d), nprocs=world, join=True)
        return [pickle.load(open(os.path.join(d, f"r{r}.pkl"), "rb")) for r in range(world)]


def single(name, gq, gaux, nx, ny, dx, dy, order, limiter, bc, steps):
    q = gq.copy(order="F")
    aux = gaux.copy(order="F") if gaux is not None else None
    s = O.make_solver(name, **PARAMS[name])
    reps, err = [], None
    for _ in range(steps):
        try:
            r = O.step(q, aux, O.Spec(nx, ny, dx, dy), s, O.Controller(0.9), bc_x=bc, bc_y=bc,
                       order=order, limiter=limiter)
        except O.OracleError as e:
            err = e
            break
        reps.append((r.dt, r.max_speed_x, r.max_speed_y))
    return q, reps, err


def test_row_strips_partition():
    st = PL.RowStrips(31, 3)
    assert [st.bounds(r) for r in range(3)] == [(0, 11), (11, 21), (21, 31)]
    assert st.neighbours(0, False) == (None, 1)
    assert st.neighbours(2, True) == (1, 0)
    assert st.neighbours(0, True) == (2, 1)
    assert PL.RowStrips(4, 2).neighbours(0, True) == (1, 1)
    with pytest.raises(ValueError):
        PL.RowStrips(5, 3)


@pytest.mark.parametrize("world,name,order,limiter,bc", [
    (2, "shallow-water-roe", 2, "mc", "extrapolate"),
    (2, "euler-hlle", 2, "minmod", "periodic"),
    (3, "euler-hlle", 2, "superbee", "periodic"),
    (3, "acoustics-var", 2, "mc", "extrapolate"),
    (2, "euler", 1, "none", "periodic"),
])
def test_n_rank_run_is_bitwise_the_single_domain_run(world, name, order, limiter, bc):
    nx, ny, steps = 20, 31, 4
    dx, dy = 1 / nx, 1 / ny
    gq, gaux = random_state(name, nx, ny, 5)
    ref_q, ref_reps, _ = single(name, gq, gaux, nx, ny, dx, dy, order, limiter, bc, steps)
    parts = run_sharded(world, name, gq, gaux, nx, ny, dx, dy, order, limiter, bc, steps)
    for p in parts:
        assert p["reports"] == ref_reps
        assert p["error"] is None
        assert np.array_equal(p["q"], ref_q[:, 2:-2, 2 + p["j0"]:2 + p["j1"]])


def test_inadmissible_cell_on_one_rank_stops_every_rank():
    name, nx, ny = "shallow-water-roe", 16, 20
    gq, _ = random_state(name, nx, ny, 6)
    gq[0, 2 + 7, 2 + 15] = -1.0          # row 15 lives on rank 1 of 2
    _, _, err = single(name, gq, None, nx, ny, 1 / nx, 1 / ny, 2, "mc", "extrapolate", 2)
    assert err is not None
    parts = run_sharded(2, name, gq, None, nx, ny, 1 / nx, 1 / ny, 2, "mc", "extrapolate", 2)
    keys = {p["error"] for p in parts}
    assert len(keys) == 1 and None not in keys
    k = keys.pop()
    d, i, j = k >> 62, (k >> 18) & 0x7FFFF, k & 0x3FFFF
    assert f"{'xy'[d]}-interface (i={i}, j={j})" == str(err).split(":")[0]


def _order_worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny = 12, 10
    q, aux = random_state("shallow-water-roe", nx, ny, 3)
    strips = PL.RowStrips(ny, world)
    sh = NumpyShard(q, aux, strips, rank, "shallow-water-roe", nx, 1 / nx, 1 / ny, 2, "mc",
                    "extrapolate")
    for _ in range(2):
        PL.sharded_step(dist, sh, strips, rank, False, 0.9)
    with open(os.path.join(outdir, f"o{rank}.pkl"), "wb") as f:
        pickle.dump(sh.calls, f)
    dist.destroy_process_group()


def test_interior_update_is_issued_while_the_halo_travels():
    """North-star overlap: after the boundary tile rows, the new rows are
    posted, the interior update is issued, and only then does the rank wait
    for the received rows; the first step primes the current state's rows."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_order_worker, args=(2, free_port(), d), nprocs=2, join=True)
        calls = [pickle.load(open(os.path.join(d, f"o{r}.pkl"), "rb")) for r in range(2)]
    for c in calls:
        assert c == ["halo_views:current", "halo_wait",
                     "update:boundary", "halo_views:next", "update:interior", "halo_wait",
                     "update:boundary", "halo_views:next", "update:interior", "halo_wait"], c
