"""Row-strip domain decomposition across GPUs (north_star subsystem 4).

The reference has no domain decomposition (a non-goal); the
north star asks for row strips along j with 2-cell halos, the exchange
overlapped with the interior tile computation.  Each rank owns global rows
[j0, j1) (ny/P each, the remainder to the first ranks) and runs one C-ABI
handle on its GPU.  Per time step (host collectives, NCCL):

  1. ws_phase_speeds — local CFL max + admissibility key into a 3 x u64 slot
     (the ghost rows of the current state are already in place);
  2. all_reduce(slot, MAX) — speeds are non-negative IEEE bit patterns and
     the slot stores NKEY_MAX - key, so int64 MAX gives the global max speed
     and the globally first inadmissible interface (reference order);
  3. ws_phase_update_part 1 — every rank computes the identical dt and
     updates the boundary tile rows (every row a neighbour needs);
  4. halo exchange of the NEW state — its first/last two rows of every
     component go to the neighbours' ghost rows (one contiguous block each
     way: the SoA row layout makes 2 rows x all components contiguous), with
     periodic y and P > 1 ranks 0 and P-1 are neighbours — while
  5. ws_phase_update_part 2 updates the interior tile rows; the next step's
     pre-pass waits for the received rows.

The first step after an upload exchanges the current state's rows once.
Because the max is order independent and the update is local, an N-rank run
is bitwise identical to the 1-GPU run (the reference's serial-twin guard,
bench.py:181-185, becomes the 1-vs-N test).  The opt-in device collectives
(``--device-reduce`` / ``--device-halo``) move steps 2 and 4 into the
kernels over peer memory.

The orchestration is generic over a *shard executor*: ``CudaShard`` (the
product: device buffers borrowed from torch, NCCL collectives) or any test
double with the same methods (tests use a numpy one over gloo).
"""

from __future__ import annotations

import contextlib
import json
import os
import statistics
import time
from dataclasses import dataclass

import numpy as np

from . import _abi

NKEY_MAX = (1 << 63) - 1


@dataclass(frozen=True)
class RowStrips:
    """Contiguous row strips along y; remainder rows go to the first ranks."""

    ny: int
    nranks: int

    def __post_init__(self):
        if self.nranks < 1 or self.ny < 2 * self.nranks:
            raise ValueError(f"need at least 2 rows per rank, got ny={self.ny}, "
                             f"ranks={self.nranks}")

    def bounds(self, rank: int) -> tuple[int, int]:
        base, extra = divmod(self.ny, self.nranks)
        j0 = rank * base + min(rank, extra)
        return j0, j0 + base + (1 if rank < extra else 0)

    def neighbours(self, rank: int, periodic: bool) -> tuple[int | None, int | None]:
        lo = rank - 1 if rank > 0 else (self.nranks - 1 if periodic and self.nranks > 1 else None)
        hi = rank + 1 if rank < self.nranks - 1 else (0 if periodic and self.nranks > 1 else None)
        return lo, hi

    def row_modes(self, rank: int, periodic: bool) -> tuple[int, int]:
        """ws_rowmode of the bottom / top ghost rows of `rank`."""
        lo, hi = self.neighbours(rank, periodic)
        return (_abi.ROWS_MEMORY if lo is not None else _abi.ROWS_BC,
                _abi.ROWS_MEMORY if hi is not None else _abi.ROWS_BC)


def periodic_rows(bc: str) -> bool:
    return bc == "periodic"


def shard_block(global_field: np.ndarray, j0: int, j1: int) -> np.ndarray:
    """Rows [j0-2, j1+2) of a global (ncomp, nx+4, ny+4) F-order field: the
    shard's host block, its ghost rows being the neighbours' interior rows."""
    return np.asfortranarray(global_field[:, :, j0:j1 + 4])


def exchange_halos(dist, shard, strips: RowStrips, rank: int, periodic: bool, group=None,
                   which: str = "current"):
    """Send the 2 boundary rows to each neighbour, receive its rows into ghosts."""
    finish_halos(shard, post_halos(dist, shard, strips, rank, periodic, group, which))


def finish_halos(shard, reqs):
    for req in reqs:
        req.wait()
    shard.halo_received()


def post_halos(dist, shard, strips: RowStrips, rank: int, periodic: bool, group=None,
               which: str = "current"):
    """Issue the halo sends/receives of the current state buffer, or of the
    next one (the state the running update writes); returns the requests
    (finish_halos waits)."""
    lo, hi = strips.neighbours(rank, periodic)
    send_lo, send_hi, recv_lo, recv_hi = shard.halo_views(which)
    # Fixed per-peer order (NCCL matches point-to-point ops to one peer in
    # issue order; with periodic P == 2 both neighbours are the same rank):
    # top rows go up first (tag 1, they land in the upper neighbour's recv_lo),
    # then bottom rows go down (tag 2, into the lower neighbour's recv_hi).
    ops = []
    if hi is not None:
        ops.append(dist.P2POp(dist.isend, send_hi, hi, group=group, tag=1))
    if lo is not None:
        ops.append(dist.P2POp(dist.isend, send_lo, lo, group=group, tag=2))
    if lo is not None:
        ops.append(dist.P2POp(dist.irecv, recv_lo, lo, group=group, tag=1))
    if hi is not None:
        ops.append(dist.P2POp(dist.irecv, recv_hi, hi, group=group, tag=2))
    return dist.batch_isend_irecv(ops) if ops else []


def sharded_step(dist, shard, strips: RowStrips, rank: int, periodic: bool, ctl, group=None,
                 device_reduce: bool = False, device_halo: bool = False):
    """One globally consistent time step.

    Host collectives (the default): the ghost rows of the current state are
    in place (the previous step sent them; the first step after an upload
    exchanges them once), so the pre-pass runs whole, the 3-word slot is
    MAX all-reduced, and the update runs in two launches: the boundary tile
    rows first (every row a neighbour needs), then -- while their new rows
    travel to the neighbours -- the interior tile rows.  Later work on the
    stream waits for the received rows (finish_halos).  With
    ``device_reduce`` (shards set up with ``set_peers``) the all-reduce is
    done by the kernels themselves over peer memory; with ``device_halo``
    the update kernels push the halo rows into the neighbours' buffers.
    """
    ctx = getattr(shard, "stream_context", None)
    with ctx() if ctx is not None else contextlib.nullcontext():
        if not getattr(shard, "halos_primed", True):
            # first step after an upload: the ghost rows come from the host
            # exchange once; later steps' come with the previous step
            exchange_halos(dist, shard, strips, rank, periodic, group)
            shard.halos_primed = True
        if device_halo:
            # the neighbours' update kernels store our ghost rows; part 2 of
            # the pre-pass waits for them on the device
            shard.phase_speeds_interior()
            shard.phase_speeds_boundary()
        else:
            shard.phase_speeds()
        if not device_reduce:
            slot = shard.slot_view()
            dist.all_reduce(slot, op=dist.ReduceOp.MAX, group=group)
            shard.slot_reduced()
        # (device_reduce: the pre-pass pushed the slot into every shard's and
        # the update waits for all pushes on the device — no host collective)
        if device_halo:
            shard.phase_update(ctl)
            return
        shard.phase_update_boundary(ctl)
        reqs = post_halos(dist, shard, strips, rank, periodic, group, which="next")
        shard.phase_update_interior(ctl)      # overlaps the halo transfer
        finish_halos(shard, reqs)


class StepGraph:
    """Two whole sharded steps (host collectives: NCCL all-reduce of the slot
    and the halo send/recv included) captured once into a torch CUDA graph
    and replayed, so a rank issues one graph launch per two steps instead of
    four library calls and three collectives per step.  The library's step
    and launch counts follow the replays (ws_capture_begin / _end,
    ws_replayed); two steps keep the ping-pong parity of every replay equal
    to the captured one.  Shards with device collectives (``--device-halo``)
    need no host call per step at all: they run whole steps through
    ``DeviceGrid.run`` (ws_run's own two-step graph)."""

    STEPS = 2

    def __init__(self, dist, shard, strips: RowStrips, rank: int, periodic: bool, ctl,
                 group=None, device_reduce: bool = False):
        torch = shard.torch
        self.shard = shard
        if not getattr(shard, "halos_primed", True):
            # the first step after an upload primes the ghost rows by a host
            # exchange, which is not part of the repeated step
            sharded_step(dist, shard, strips, rank, periodic, ctl, group,
                         device_reduce=device_reduce)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        shard.grid.capture_begin()
        try:
            with torch.cuda.graph(self.graph, stream=shard.torch_stream):
                for _ in range(self.STEPS):
                    sharded_step(dist, shard, strips, rank, periodic, ctl, group,
                                 device_reduce=device_reduce)
        finally:
            self.steps, self.launches = shard.grid.capture_end()

    def replay(self):
        """STEPS more steps, enqueued on the shard's stream."""
        with self.shard.stream_context():
            self.graph.replay()
        self.shard.grid.replayed(self.steps, self.launches)


def decode_slot(slot_words) -> tuple[float, float, int | None]:
    """(max_sx, max_sy, first error key or None) from the 3 reduced words."""
    bx, by, nk = (int(w) & ((1 << 64) - 1) for w in slot_words)
    sx = np.array([bx], dtype=np.uint64).view(np.float64)[0]
    sy = np.array([by], dtype=np.uint64).view(np.float64)[0]
    return float(sx), float(sy), (None if nk == 0 else NKEY_MAX - nk)


# ---------------------------------------------------------------------------
# the product executor: one GPU shard, buffers owned by torch

class CudaShard:
    """DeviceGrid shard whose state/aux/slot buffers are torch tensors, so the
    halo rows and the reduction slot can be handed to torch.distributed
    (NCCL) without copies."""

    def __init__(self, case, strips: RowStrips, rank: int, device, periodic_y: bool,
                 precision: str = "f64", stream=None, symmetric: bool = False):
        import torch

        from .device import DeviceGrid
        from .kernels import make_kernel
        self.torch = torch
        j0, j1 = strips.bounds(rank)
        self.j0, self.j1 = j0, j1
        self.ny = j1 - j0
        lo_mode, hi_mode = strips.row_modes(rank, periodic_y)
        kernel = make_kernel(case.kernel, **case.kernel_params)
        desc = _abi.WsDesc()
        desc.nx, desc.ny, desc.dx, desc.dy, desc.num_ghost = case.nx, self.ny, case.dx, case.dy, 2
        desc.solver = _abi.SOLVER_IDS[case.kernel]
        desc.order = case.order
        desc.limiter = _abi.LIMITER_IDS[case.limiter]
        desc.bc_x = desc.bc_y = _abi.BC_IDS[case.bc]
        desc.precision = _abi.PRECISION_IDS[precision]
        desc.ny_global, desc.j_offset = strips.ny, j0
        desc.rows_lo, desc.rows_hi = lo_mode, hi_mode
        import ctypes
        qb, ab, sb = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        _abi.check(_abi.lib().ws_buffer_bytes(ctypes.byref(desc), ctypes.byref(qb),
                                              ctypes.byref(ab), ctypes.byref(sb)))
        u8 = dict(dtype=torch.uint8, device=device)
        if symmetric:
            import torch.distributed._symmetric_memory as symm
            self.bufs = [symm.empty(qb.value, dtype=torch.uint8, device=device).zero_()
                         for _ in range(2)]
        else:
            self.bufs = [torch.zeros(qb.value, **u8), torch.zeros(qb.value, **u8)]
        self.aux_buf = torch.zeros(max(ab.value, 8), **u8)
        nslot = (sb.value + 7) // 8 * 8
        if symmetric:
            import torch.distributed._symmetric_memory as symm
            self.slots = symm.empty(nslot, dtype=torch.uint8, device=device)
            self.slots.zero_()
        else:
            self.slots = torch.zeros(nslot, **u8)
        self.grid = DeviceGrid(case.nx, self.ny, case.dx, case.dy, kernel, order=case.order,
                               limiter=case.limiter, bc_x=case.bc, bc_y=case.bc,
                               precision=precision, device=device.index or 0,
                               ny_global=strips.ny, j_offset=j0, rows_lo=lo_mode,
                               rows_hi=hi_mode,
                               buffers={"q0": self.bufs[0].data_ptr(),
                                        "q1": self.bufs[1].data_ptr(),
                                        "aux": self.aux_buf.data_ptr() if ab.value else None,
                                        "slots": self.slots.data_ptr()})
        # one torch stream carries the shard's kernels AND its collectives:
        # sharded_step makes it current, so NCCL (which orders itself after
        # the current stream) and the C ABI calls (given its handle) are in
        # one stream order.  A null handle would select the library's own
        # non-blocking stream, which nothing on the torch side waits for.
        self.torch_stream = stream if stream is not None else torch.cuda.Stream(device)
        self.stream = self.torch_stream.cuda_stream
        assert self.stream, "CudaShard needs a non-default torch stream"

    def stream_context(self):
        return self.torch.cuda.stream(self.torch_stream)

    def set_peers(self, state_ptrs):
        """Device-side slot reduction: DevState pointers of all shards (this
        shard's slots buffer is its DevState), as mapped on this GPU."""
        self.grid.set_peers(state_ptrs)

    def upload(self, q_block, aux_block=None):
        """Host block of this strip (ghost rows included); with device halos
        the next step primes the ghost rows through the host exchange."""
        self.grid.upload(q_block, aux_block, stream=self.stream)
        self.halos_primed = False

    def set_halo_peers(self, lo=None, hi=None):
        """Device-side halos: lo = (q0, q1, state, ny) / hi = (q0, q1, state)
        device pointers of the neighbour shards as mapped here."""
        self.grid.set_halo_peers(lo, hi)

    def enable_device_halo(self, strips, rank, periodic, group=None):
        """Symmetric-memory rendezvous of the state buffers; hand the
        neighbours' buffers and DevState to the library (the DevState table
        comes from enable_device_reduce, which must run first)."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        grp = group if group is not None else dist.group.WORLD
        h0 = symm.rendezvous(self.bufs[0], grp)
        h1 = symm.rendezvous(self.bufs[1], grp)
        hs = symm.rendezvous(self.slots, grp)
        lo, hi = strips.neighbours(rank, periodic)
        arg = lambda r: (int(h0.buffer_ptrs[r]), int(h1.buffer_ptrs[r]),  # noqa: E731
                         int(hs.buffer_ptrs[r]))
        self.set_halo_peers(None if lo is None else arg(lo) + (strips.bounds(lo)[1] -
                                                                strips.bounds(lo)[0],),
                            None if hi is None else arg(hi))

    def enable_device_reduce(self, group=None):
        """Map every rank's DevState through torch symmetric memory and hand
        the table to the library (multi-GPU, one process per GPU).  The
        shard's slots buffer must have been allocated symmetric
        (``CudaShard(..., symmetric=True)``)."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        grp = group if group is not None else dist.group.WORLD
        hdl = symm.rendezvous(self.slots, grp)
        ptrs = [int(hdl.buffer_ptrs[r]) for r in range(hdl.world_size)]
        self.set_peers(ptrs)

    def _current(self, which="current"):
        ptr, pitch, row = self.grid.state_ptr()
        k = 0 if ptr == self.bufs[0].data_ptr() else 1
        if which == "next":
            k ^= 1
        return self.bufs[k], row * (8 if self.grid.precision == "f64" else 4)

    def halo_views(self, which="current"):
        """(send_lo, send_hi, recv_lo, recv_hi) byte views of the current state
        buffer, or of the next one (the state the running update writes)."""
        buf, rbytes = self._current(which)
        n = self.ny
        return (buf[2 * rbytes:4 * rbytes], buf[n * rbytes:(n + 2) * rbytes],
                buf[0:2 * rbytes], buf[(n + 2) * rbytes:(n + 4) * rbytes])

    def halo_received(self):
        pass

    def phase_speeds(self):
        self.grid.phase_speeds(stream=self.stream)

    def phase_speeds_interior(self):
        """Pre-pass edges that do not read the ghost rows being received."""
        self.grid.phase_speeds(stream=self.stream, part=1)

    def phase_speeds_boundary(self):
        """The y-edges that read the received ghost rows (row 0, periodic row ny)."""
        self.grid.phase_speeds(stream=self.stream, part=2)

    def slot_view(self):
        off = self.grid.slot_ptr() - self.slots.data_ptr()
        return self.slots[off:off + 24].view(self.torch.int64)

    def slot_reduced(self):
        pass

    def phase_update(self, ctl):
        self.grid.phase_update(ctl, stream=self.stream)

    def phase_update_boundary(self, ctl):
        """Update part 1: the tile rows holding the rows the neighbours need."""
        self.grid.phase_update(ctl, stream=self.stream, part=1)

    def phase_update_interior(self, ctl):
        """Update part 2: the interior tile rows (overlaps the halo transfer)."""
        self.grid.phase_update(ctl, stream=self.stream, part=2)


# ---------------------------------------------------------------------------
# bench.py --gpus N (torchrun): weak (default) or strong scaling

def rank_strip(args, rank, world, strong, build_case, dev):
    """(case, strips, host q block, host aux block) of this rank.

    C5 (the default): only this rank's rows of the global recipe are made
    (weak: nx = 16384, ny = 16384 P with 64 P bumps; strong: the 16384^2
    grid cut in P strips), on the GPU from the host's numpy factors; other
    configs slice the 1-GPU case (weak: P stacked copies).  The ghost rows a
    neighbour owns are primed by the first step's exchange; aux (never
    exchanged) carries its neighbour rows here."""
    from . import configs
    size = getattr(args, "size", None)
    prec = args.precision or "f64"
    if args.config == "c5":
        n = size or 16384
        ny_g = n if strong else n * world
        strips = RowStrips(ny_g, world)
        j0, j1 = strips.bounds(rank)
        case = configs.c5_bumps(n, ny=ny_g, rows=(j0, j1), dtype=prec, device=dev)
        h = case.meta.pop("h_dev").t().contiguous().cpu().numpy()
        q = configs._field(3, n, j1 - j0)
        q[0, 2:-2, 2:-2] = h
        case.name = "C5-shallow-water-scaling"
        return case, strips, q, None
    base = build_case(args.config, precision=args.precision, device=dev, size=size)
    ny_g = base.ny if strong else base.ny * world
    strips = RowStrips(ny_g, world)
    j0, j1 = strips.bounds(rank)

    def block(f):
        if f is None:
            return None
        inner = f[:, :, 2:-2]
        if strong:
            g = f.copy(order="F")
        else:   # P copies stacked along y
            g = np.zeros((f.shape[0], base.nx + 4, ny_g + 4), order="F")
            for r in range(world):
                g[:, :, 2 + r * base.ny:2 + (r + 1) * base.ny] = inner
        if periodic_rows(base.bc):
            g[:, :, 0:2] = g[:, :, ny_g:ny_g + 2]
            g[:, :, ny_g + 2:ny_g + 4] = g[:, :, 2:4]
        return shard_block(g, j0, j1)

    return base, strips, block(base.q), block(base.aux)


def bench_sharded(args, rank, world, local, build_case, Clocks, cpu_rate, peak_fn, METRIC, UNIT,
                  workload_config=None, cpu_baseline=None):
    import torch
    import torch.distributed as dist

    from . import configs
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    os.environ.setdefault("RANK", str(rank))
    os.environ.setdefault("WORLD_SIZE", str(world))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    strong = bool(getattr(args, "strong", False))
    case, strips, q_block, aux_block = rank_strip(args, rank, world, strong, build_case, dev)
    prec = args.precision or case.dtype
    ny_g = strips.ny
    j0, j1 = strips.bounds(rank)
    periodic = case.bc == "periodic"
    dhalo = bool(getattr(args, "device_halo", False))
    dred = bool(getattr(args, "device_reduce", False)) or dhalo
    shard = CudaShard(case, strips, rank, dev, periodic, prec, symmetric=dred)
    if dred:
        shard.enable_device_reduce()
    if dhalo:
        shard.enable_device_halo(strips, rank, periodic)
    npdt = np.float64 if prec == "f64" else np.float32
    host_q = np.asfortranarray(q_block, dtype=npdt)
    host_aux = np.asfortranarray(aux_block, dtype=npdt) if aux_block is not None else None
    del q_block, aux_block
    shard.upload(host_q, host_aux)
    if dred:
        torch.cuda.synchronize()
        dist.barrier()      # every arrival counter reset before the first push
    ctl = _abi.make_ctl(case.cfl)
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        sharded_step(dist, shard, strips, rank, periodic, ctl, device_reduce=dred,
                     device_halo=dhalo)
    torch.cuda.synchronize()
    res = shard.grid.poll()
    shard.grid.raise_for(res.error)
    k = args.steps
    # the default issue path: whole steps from graphs (device collectives:
    # ws_run's own; host collectives: a captured StepGraph of two steps with
    # the NCCL calls inside); --eager issues every step from Python
    # (a strip whose state fits twice in the 126 MB L2 steps eagerly: the L2
    # is flushed between its timed steps, which a replayed graph would not do)
    esz = 8 if prec == "f64" else 4
    strip_bytes = host_q.shape[0] * case.nx * (j1 - j0) * esz
    eager = bool(getattr(args, "eager", False)) or strip_bytes < (256 << 20)
    whole = dhalo and dred
    sgraph = None
    graph_note = None
    if not eager and not whole:
        try:
            sgraph = StepGraph(dist, shard, strips, rank, periodic, ctl, device_reduce=dred)
        except Exception as e:  # noqa: BLE001 - capture of the NCCL P2P calls refused
            # (verified at world size 1 only): every rank steps eagerly instead
            graph_note = f"graph capture failed ({type(e).__name__}: {e}); eager"
        ok = torch.tensor([0 if sgraph is None else 1], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            sgraph = None
            eager = True
            graph_note = graph_note or "graph capture failed on another rank; eager"

    def graph_steps(n):
        """n steps from graphs (one eager step when n is odd)."""
        if whole:
            shard.grid.run(n, ctl, stream=shard.stream)
            return
        for _ in range(n // 2):
            sgraph.replay()
        if n % 2:
            sharded_step(dist, shard, strips, rank, periodic, ctl, device_reduce=dred)

    def timed_graph():
        """k steps from graphs, one event pair around them (device time)."""
        e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        dist.barrier()
        torch.cuda.synchronize()
        with shard.stream_context():
            torch.cuda._sleep(int(2e6))
            flush.zero_()
            e0.record()
            graph_steps(k)
            e1.record()
            torch.cuda.synchronize()
        dist.barrier()
        return e0.elapsed_time(e1)

    def timed(split):
        """k steps; split: events also around the update (parts 1 + 2)."""
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(k)]
        dist.barrier()
        torch.cuda.synchronize()
        with shard.stream_context():
            # queued GPU sleep: the host enqueues the whole loop (every op is
            # asynchronous, NCCL included) so event gaps are device time;
            # flush, events, kernels and collectives on the shard's stream
            torch.cuda._sleep(int(2e6 + 6e5 * k))
            for i in range(k):
                flush.zero_()
                evs[i][0].record()
                if split and not dhalo:
                    shard.phase_speeds()
                    if not dred:
                        dist.all_reduce(shard.slot_view(), op=dist.ReduceOp.MAX)
                    evs[i][1].record()
                    shard.phase_update_boundary(ctl)
                    reqs = post_halos(dist, shard, strips, rank, periodic, which="next")
                    shard.phase_update_interior(ctl)
                    evs[i][2].record()
                    finish_halos(shard, reqs)
                else:
                    sharded_step(dist, shard, strips, rank, periodic, ctl, device_reduce=dred,
                                 device_halo=dhalo)
                evs[i][3].record()
            torch.cuda.synchronize()
        dist.barrier()
        return evs

    l0 = shard.grid.launches()
    with Clocks(local) as clk:
        if eager:
            evs = timed(False)
            ms = sum(e[0].elapsed_time(e[3]) for e in evs)
        else:
            ms = timed_graph()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    res = shard.grid.poll()
    shard.grid.raise_for(res.error)
    launches = shard.grid.launches() - l0
    cells = case.nx * ny_g
    value = cells * k / (ms_max / 1e3)
    upd_ms = None
    if not dhalo:
        # the dominant kernel: the update (boundary + interior launches, the
        # halo sends enqueued between them), event-timed in a second loop
        evs = timed(True)
        upd_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
        res = shard.grid.poll()
        shard.grid.raise_for(res.error)
    e2e = None
    if not getattr(args, "no_e2e", False):
        e2e = sharded_e2e(dist, shard, strips, rank, periodic, ctl, host_q, host_aux, k, cells,
                          UNIT, dev, dred, dhalo)
    if rank == 0:
        peak, kind = peak_fn()
        bpc = configs.bytes_per_cell(case.kernel, prec)
        local_cells = case.nx * (j1 - j0)
        t_kernel = upd_ms if upd_ms else ms_max / k
        achieved = local_cells * bpc / (t_kernel / 1e3) / 1e9
        cfg = (workload_config(case, world, strong, ny_total=ny_g) if workload_config else
               {"workload": case.name, "nx": case.nx, "ny": ny_g})
        cpu = None
        if world == 1 and cpu_baseline is not None and not getattr(args, "no_cpu", False):
            cpu = cpu_baseline(args.config, args, precision=args.precision,
                               size=getattr(args, "size", None))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": k,
            "warmup": args.warmup, "ms_per_step": ms_max / k, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": prec,
            "data": "synthetic",
            "config": cfg,
            "measurement": {
                "parallelism": f"row-strips{world}",
                "issue": (graph_note if graph_note else
                          "every step from Python (--eager)" if eager else
                          "ws_run's two-step graph per rank (device collectives)" if whole else
                          "a captured torch CUDA graph of two steps per rank (NCCL calls "
                          "inside), replayed; the strip's state is larger than the L2"),
                "timed_step": ("CFL pre-pass + update with halo rows and the slot reduction "
                               "done by the kernels over peer memory") if dhalo else
                              ("CFL pre-pass + device-side slot reduction over peer memory + "
                               "update (boundary tile rows, halo sends, interior tile rows)")
                              if dred else
                              "CFL pre-pass + MAX all-reduce + update (boundary tile rows, "
                              "then the interior tile rows while the new halo rows travel)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": ("k_update_w (boundary + interior launches), rank 0"
                                    if upd_ms else "whole step"),
                         "kernel_ms": t_kernel, "peak_kind": kind,
                         "algorithmic_bytes_per_cell": bpc},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    shard.grid.close()
    dist.destroy_process_group()
    return 0


def sharded_e2e(dist, shard, strips, rank, periodic, ctl, host_q, host_aux, k, cells, unit, dev,
                dred=False, dhalo=False):
    """Whole-job e2e at N ranks through the public API: per step every rank
    uploads its strip from pinned host memory, the sharded step runs, every
    rank downloads its strip; wall time max over ranks."""
    import torch
    pin = lambda a: (None if a is None else  # noqa: E731
                     torch.from_numpy(np.ascontiguousarray(a.ravel(order="F")))
                     .pin_memory().numpy().reshape(a.shape, order="F"))
    pq, pa = pin(host_q), pin(host_aux)
    out = pin(np.zeros_like(host_q))
    n = max(3, min(k, 10))
    def one():
        shard.upload(pq, pa)
        if dred:
            # every rank's upload resets its arrival counter before anyone pushes
            torch.cuda.synchronize()
            dist.barrier()
        sharded_step(dist, shard, strips, rank, periodic, ctl, device_reduce=dred,
                     device_halo=dhalo)
        shard.grid.download(out, stream=shard.stream)

    for _ in range(2):
        one()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(n):
        one()
    el = time.perf_counter() - t0
    t = torch.tensor([el], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    res = shard.grid.poll()
    shard.grid.raise_for(res.error)
    hb = pq.nbytes + (pa.nbytes if pa is not None else 0)
    return {"value": cells * n / float(t.item()), "unit": unit,
            "h2d_bytes_per_step": hb * dist.get_world_size(),
            "d2h_bytes_per_step": out.nbytes * dist.get_world_size(),
            "api": "per rank: DeviceGrid.upload(strip) / sharded_step / DeviceGrid.download "
                   "(pinned host), wall time max over ranks"}
