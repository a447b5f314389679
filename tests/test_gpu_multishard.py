"""Row-strip shards on ONE GPU (no NCCL, nothing waits on another kernel):
P CudaShard handles with torch-owned buffers; halo rows are moved with
torch copies and the 3-word slot is max-reduced with torch — the same data
flow sharded_step runs over NCCL.  Must equal the single-domain oracle
bitwise (state of every shard, every dt), including periodic wrap-around
between the first and last strip and an inadmissible cell on one strip."""

from types import SimpleNamespace

import numpy as np
import pytest

from helpers import PARAMS, oracle_run, random_state
from oracle import wavestep_oracle as O

pytestmark = pytest.mark.gpu


def fake_sharded(name, gq, gaux, nx, ny, dx, dy, P, steps, order, limiter, bc,
                 device_reduce=False, device_halo=False, inspect=None, split_update=False):
    import torch

    from paper_1308_1464_b200 import _abi
    from paper_1308_1464_b200 import parallel as PL
    dev = torch.device("cuda", 0)
    case = SimpleNamespace(kernel=name, kernel_params=PARAMS[name], nx=nx, dx=dx, dy=dy,
                           order=order, limiter=limiter, bc=bc)
    periodic = bc == "periodic"
    # the global ghost frame as the single domain sees it (static aux rows of
    # a periodic strip boundary included)
    gq = np.asfortranarray(gq.copy())
    O.fill_ghost(gq, bc, bc)
    if gaux is not None:
        gaux = np.asfortranarray(gaux.copy())
        O.fill_ghost(gaux, bc, bc)
    strips = PL.RowStrips(ny, P)
    # one shared stream: the torch copies standing in for NCCL are ordered
    # with every shard's kernels
    stream = torch.cuda.Stream(dev)
    shards = [PL.CudaShard(case, strips, r, dev, periodic, stream=stream) for r in range(P)]
    for r, sh in enumerate(shards):
        j0, j1 = strips.bounds(r)
        sh.grid.upload(PL.shard_block(gq, j0, j1),
                       PL.shard_block(gaux, j0, j1) if gaux is not None else None,
                       stream=sh.stream)
    if device_reduce:
        # every shard's DevState (its slots buffer) in every shard's table:
        # the pre-passes push their slots, the updates wait for P arrivals
        ptrs = [sh.slots.data_ptr() for sh in shards]
        for sh in shards:
            sh.set_peers(ptrs)
    if device_halo:
        # each shard's update stores its boundary rows into the neighbours'
        # ghost rows; their pre-pass part 2 waits for the pushes
        for r, sh in enumerate(shards):
            lo, hi = strips.neighbours(r, periodic)
            info = lambda k: (shards[k].bufs[0].data_ptr(), shards[k].bufs[1].data_ptr(),  # noqa: E731
                              shards[k].slots.data_ptr())
            sh.set_halo_peers(None if lo is None else info(lo) + (shards[lo].ny,),
                              None if hi is None else info(hi))
    ctl = _abi.make_ctl(0.9)
    torch.cuda.set_stream(stream)

    def copy_halos(which):
        views = [sh.halo_views(which) for sh in shards]
        for r in range(P):
            lo, hi = strips.neighbours(r, periodic)
            if hi is not None:
                views[hi][2].copy_(views[r][1])
            if lo is not None:
                views[lo][3].copy_(views[r][0])

    def reduce_slots():
        slot = shards[0].slot_view().clone()
        for sh in shards[1:]:
            slot = torch.maximum(slot, sh.slot_view())
        for sh in shards:
            sh.slot_view().copy_(slot)

    if split_update:
        # the product's sharded_step order: prime the current rows once; per
        # step the whole pre-pass, the slot reduction, the boundary tile rows,
        # the NEW state's rows to the neighbours, then the interior tile rows
        copy_halos("current")
        for it in range(steps):
            for sh in shards:
                sh.phase_speeds()
            reduce_slots()
            for sh in shards:
                sh.phase_update_boundary(ctl)
            copy_halos("next")
            for sh in shards:
                sh.phase_update_interior(ctl)
        steps = 0
    for it in range(steps):
        # part 1 of the pre-pass runs BEFORE the halo rows are refreshed (the
        # ghost rows still hold the previous step's values): it must not read them
        for sh in shards:
            sh.phase_speeds_interior()
        if not device_halo or it == 0:
            # (device halos: the first step's ghost rows are primed by a copy;
            # later ones are pushed by the neighbours' update kernels)
            views = [sh.halo_views() for sh in shards]
            for r in range(P):
                lo, hi = strips.neighbours(r, periodic)
                if hi is not None:
                    views[hi][2].copy_(views[r][1])  # my top rows -> upper neighbour's low ghosts
                if lo is not None:
                    views[lo][3].copy_(views[r][0])  # my bottom rows -> lower neighbour's high ghosts
        for sh in shards:
            sh.phase_speeds_boundary()
        if not device_reduce:
            slot = shards[0].slot_view().clone()
            for sh in shards[1:]:
                slot = torch.maximum(slot, sh.slot_view())
            for sh in shards:
                sh.slot_view().copy_(slot)
        for sh in shards:
            sh.phase_update(ctl)
    torch.cuda.synchronize()
    torch.cuda.set_stream(torch.cuda.default_stream(dev))
    out, reps, errs = [], [], []
    for sh in shards:
        res = sh.grid.poll()
        reps.append([r[0] for r in res.reports])
        errs.append(res.error)
        out.append(sh.grid.download()[:, 2:-2, 2:-2])
        if inspect is not None:
            inspect(sh.grid)
        sh.grid.close()
    return out, reps, errs, strips


@pytest.mark.parametrize("name,P,bc", [("shallow-water-roe", 2, "extrapolate"),
                                       ("shallow-water-roe", 3, "periodic"),
                                       ("euler-hlle", 3, "periodic"),
                                       ("acoustics-var", 4, "extrapolate"),
                                       ("euler", 2, "periodic")])
def test_split_update_overlap_order_bitwise(name, P, bc):
    # boundary tile rows -> halo rows of the new state -> interior tile rows
    # (the host-collective sharded_step): bitwise the single-domain oracle;
    # the strips (ny = 100 over P) hold 1 to 4 tile rows, so part 2 is empty
    # on some and the step's CTA count spans both launches
    nx, ny, steps = 83, 100, 4
    dx, dy = 1.0 / nx, 1.0 / ny
    q, aux = random_state(name, nx, ny, 12)
    oq, oreps = oracle_run(name, q, aux, nx, ny, dx, dy, steps=steps, order=2, limiter="mc",
                           bc_x=bc, bc_y=bc)
    out, reps, errs, strips = fake_sharded(name, q, aux, nx, ny, dx, dy, P, steps, 2, "mc", bc,
                                           split_update=True)
    assert all(e.code == 0 for e in errs)
    for r in reps:
        assert r == [x.dt for x in oreps]
    assert np.array_equal(np.concatenate(out, axis=2), oq[:, 2:-2, 2:-2])


@pytest.mark.parametrize("name,P,bc,order,limiter", [
    ("shallow-water-roe", 2, "extrapolate", 2, "mc"),
    ("shallow-water-roe", 3, "periodic", 2, "superbee"),
    ("euler-hlle", 2, "periodic", 2, "minmod"),
    ("acoustics-var", 3, "extrapolate", 2, "mc"),
    ("acoustics-const", 2, "periodic", 1, "none"),
    ("euler", 4, "extrapolate", 1, "none"),
])
def test_fake_shards_bitwise_single_domain(name, P, bc, order, limiter):
    nx, ny, steps = 45, 70, 5
    dx, dy = 1 / nx, 1 / ny
    gq, gaux = random_state(name, nx, ny, 21)
    ref, oreps = oracle_run(name, gq, gaux, nx, ny, dx, dy, steps=steps, order=order,
                            limiter=limiter, bc_x=bc, bc_y=bc)
    out, reps, errs, strips = fake_sharded(name, gq, gaux, nx, ny, dx, dy, P, steps, order,
                                           limiter, bc)
    for r in range(P):
        j0, j1 = strips.bounds(r)
        assert errs[r].code == 0
        assert reps[r] == [o.dt for o in oreps]
        assert np.array_equal(out[r], ref[:, 2:-2, 2 + j0:2 + j1]), f"shard {r}"


def test_fake_shards_report_the_global_first_error():
    from paper_1308_1464_b200 import _abi
    name, nx, ny = "shallow-water-roe", 20, 24
    gq, _ = random_state(name, nx, ny, 22)
    gq[0, 2 + 7, 2 + 19] = -1.0            # lives on strip 2 of 3
    with pytest.raises(O.OracleError) as oe:
        oracle_run(name, gq, None, nx, ny, 1 / nx, 1 / ny, steps=1, order=2, limiter="mc")
    _, _, errs, _ = fake_sharded(name, gq, None, nx, ny, 1 / nx, 1 / ny, 3, 1, 2, "mc",
                                 "extrapolate")
    for e in errs:
        assert e.code == _abi.WS_ERR_KERNEL
        assert f"{'xy'[e.direction]}-interface (i={e.i}, j={e.j})" == str(oe.value).split(":")[0]


def test_split_prepass_needs_a_prepass():
    # single-domain constant-coefficient acoustics has static speeds (no
    # pre-pass at all): asking for half of one is a configuration error
    from helpers import device_grid
    g = device_grid("acoustics-const", 16, 16, 1 / 16, 1 / 16)
    try:
        with pytest.raises(ValueError, match="split CFL pre-pass"):
            g.phase_speeds(part=1)
        with pytest.raises(ValueError, match="part must be"):
            g.phase_speeds(part=3)
    finally:
        g.close()


@pytest.mark.parametrize("name,P,bc,halo", [("shallow-water-roe", 3, "periodic", False),
                                            ("euler-hlle", 2, "extrapolate", False),
                                            ("acoustics-var", 4, "extrapolate", False),
                                            ("shallow-water-roe", 3, "periodic", True),
                                            ("shallow-water-roe", 2, "periodic", True),
                                            ("euler-hlle", 4, "extrapolate", True),
                                            ("acoustics-var", 3, "periodic", True)])
def test_device_side_reduction_bitwise(name, P, bc, halo):
    # ws_set_peers: no host collective at all — the pre-pass kernels push
    # their slots into every shard's and the updates wait for all pushes
    nx, ny, steps = 45, 70, 5
    dx, dy = 1 / nx, 1 / ny
    gq, gaux = random_state(name, nx, ny, 27)
    ref, oreps = oracle_run(name, gq, gaux, nx, ny, dx, dy, steps=steps, order=2,
                            limiter="mc", bc_x=bc, bc_y=bc)
    out, reps, errs, strips = fake_sharded(name, gq, gaux, nx, ny, dx, dy, P, steps, 2, "mc",
                                           bc, device_reduce=True, device_halo=halo)
    for r in range(P):
        j0, j1 = strips.bounds(r)
        assert errs[r].code == 0
        assert reps[r] == [o.dt for o in oreps]
        assert np.array_equal(out[r], ref[:, 2:-2, 2 + j0:2 + j1]), f"shard {r}"


def test_device_side_reduction_reports_the_global_first_error():
    from paper_1308_1464_b200 import _abi
    name, nx, ny = "shallow-water-roe", 20, 24
    gq, _ = random_state(name, nx, ny, 22)
    gq[0, 2 + 7, 2 + 19] = -1.0            # lives on strip 2 of 3
    with pytest.raises(O.OracleError) as oe:
        oracle_run(name, gq, None, nx, ny, 1 / nx, 1 / ny, steps=1, order=2, limiter="mc")
    _, _, errs, _ = fake_sharded(name, gq, None, nx, ny, 1 / nx, 1 / ny, 3, 1, 2, "mc",
                                 "extrapolate", device_reduce=True)
    for e in errs:
        assert e.code == _abi.WS_ERR_KERNEL
        assert f"{'xy'[e.direction]}-interface (i={e.i}, j={e.j})" == str(oe.value).split(":")[0]


def test_set_peers_validation():
    from helpers import device_grid
    g = device_grid("acoustics-const", 16, 16, 1 / 16, 1 / 16)
    try:
        with pytest.raises(ValueError, match="device-side reduction needs"):
            g.set_peers([g.devstate_ptr()])
        with pytest.raises(ValueError, match="npeers must lie"):
            g.set_peers([g.devstate_ptr()] * 9)
    finally:
        g.close()


def test_shard_refuses_whole_steps_without_device_collectives():
    import torch
    from paper_1308_1464_b200 import _abi
    from paper_1308_1464_b200 import parallel as PL
    name, nx, ny = "shallow-water-roe", 20, 24
    gq, _ = random_state(name, nx, ny, 5)
    case = SimpleNamespace(kernel=name, kernel_params=PARAMS[name], nx=nx, dx=1 / nx,
                           dy=1 / ny, order=2, limiter="mc", bc="extrapolate")
    strips = PL.RowStrips(ny, 2)
    sh = PL.CudaShard(case, strips, 0, torch.device("cuda", 0), False)
    try:
        sh.upload(PL.shard_block(gq, *strips.bounds(0)))
        with pytest.raises(ValueError, match="row-strip shard steps through"):
            sh.grid.step(_abi.make_ctl(0.9))
        with pytest.raises(ValueError, match="row-strip shard steps through"):
            sh.grid.run(3, _abi.make_ctl(0.9))
    finally:
        sh.grid.close()


@pytest.mark.parametrize("bc,dred,dhalo", [("extrapolate", False, False),
                                           ("periodic", False, False),
                                           ("periodic", True, False),
                                           ("extrapolate", True, True),
                                           ("periodic", True, True)])
def test_fake_shards_tile_prepass_skips_tiles(bc, dred, dhalo):
    # shallow water strips large enough that most tiles are skipped by the
    # tile pre-pass (the maximum sits on one dam's front), the boundary tile
    # rows next to ghost rows in memory always probed
    name, nx, ny, P, steps = "shallow-water-roe", 200, 300, 3, 8
    dx, dy = 1 / nx, 1 / ny
    rng = np.random.default_rng(4)
    gq = np.zeros((3, nx + 4, ny + 4), order="F")
    xx, yy = np.meshgrid((np.arange(nx) + 0.5) * dx, (np.arange(ny) + 0.5) * dy, indexing="ij")
    gq[0, 2:-2, 2:-2] = np.where((xx - 0.5) ** 2 + (yy - 0.33) ** 2 < 0.01, 2.0, 1.0) \
        + rng.normal(0, 1e-4, (nx, ny))
    ref, oreps = oracle_run(name, gq, None, nx, ny, dx, dy, steps=steps, order=2,
                            limiter="mc", bc_x=bc, bc_y=bc)
    out, reps, errs, strips = fake_sharded(name, gq, None, nx, ny, dx, dy, P, steps, 2, "mc", bc,
                                           device_reduce=dred, device_halo=dhalo)
    for r in range(P):
        j0, j1 = strips.bounds(r)
        assert errs[r].code == 0
        assert reps[r] == [o.dt for o in oreps]
        assert np.array_equal(out[r], ref[:, 2:-2, 2 + j0:2 + j1]), f"shard {r}"


def device_collective_shards(name, gq, gaux, nx, ny, dx, dy, P, bc, halo, order=2, limiter="mc"):
    """P shards on one GPU, each on its OWN stream, with device collectives
    (slot reduction, and halo pushes when `halo`): whole steps need no host
    collective, so ws_run replays its two-step graph per shard and the
    shards' kernels wait on one another's counters while running
    concurrently (tiny grids: every CTA of every shard is resident at once)."""
    import torch

    from paper_1308_1464_b200 import parallel as PL
    dev = torch.device("cuda", 0)
    case = SimpleNamespace(kernel=name, kernel_params=PARAMS[name], nx=nx, dx=dx, dy=dy,
                           order=order, limiter=limiter, bc=bc)
    periodic = bc == "periodic"
    gq = np.asfortranarray(gq.copy())
    O.fill_ghost(gq, bc, bc)
    if gaux is not None:
        gaux = np.asfortranarray(gaux.copy())
        O.fill_ghost(gaux, bc, bc)
    strips = PL.RowStrips(ny, P)
    shards = [PL.CudaShard(case, strips, r, dev, periodic) for r in range(P)]
    for r, sh in enumerate(shards):
        j0, j1 = strips.bounds(r)
        # the host block carries the neighbours' rows: ghost rows primed
        sh.upload(PL.shard_block(gq, j0, j1),
                  PL.shard_block(gaux, j0, j1) if gaux is not None else None)
    ptrs = [sh.slots.data_ptr() for sh in shards]
    for sh in shards:
        sh.set_peers(ptrs)
    if halo:
        for r, sh in enumerate(shards):
            lo, hi = strips.neighbours(r, periodic)
            info = lambda k: (shards[k].bufs[0].data_ptr(), shards[k].bufs[1].data_ptr(),  # noqa: E731
                              shards[k].slots.data_ptr())
            sh.set_halo_peers(None if lo is None else info(lo) + (shards[lo].ny,),
                              None if hi is None else info(hi))
    torch.cuda.synchronize()
    return shards, strips


def collect(shards):
    import torch
    torch.cuda.synchronize()
    out, reps, errs, ts = [], [], [], []
    for sh in shards:
        res = sh.grid.poll()
        reps.append([r[0] for r in res.reports])
        errs.append(res.error)
        ts.append(res.t)
        out.append(sh.grid.download()[:, 2:-2, 2:-2])
    return out, reps, errs, ts


@pytest.mark.parametrize("name,P,bc,halo", [("shallow-water-roe", 3, "periodic", True),
                                            ("euler-hlle", 2, "extrapolate", True),
                                            ("euler", 2, "periodic", True),
                                            ("acoustics-var", 3, "periodic", True)])
def test_device_collective_shards_run_from_graphs(name, P, bc, halo):
    # ws_run on every shard (10 steps: the two-step graph replayed), the
    # arrival counts awaited on the device taken from DevState::seq
    nx, ny, steps = 45, 70, 10
    dx, dy = 1 / nx, 1 / ny
    gq, gaux = random_state(name, nx, ny, 41)
    ref, oreps = oracle_run(name, gq, gaux, nx, ny, dx, dy, steps=steps, order=2,
                            limiter="mc", bc_x=bc, bc_y=bc)
    from paper_1308_1464_b200 import _abi
    shards, strips = device_collective_shards(name, gq, gaux, nx, ny, dx, dy, P, bc, halo)
    try:
        for sh in shards:
            sh.grid.run(steps, _abi.make_ctl(0.9), stream=sh.stream)
        out, reps, errs, _ = collect(shards)
        for r in range(P):
            j0, j1 = strips.bounds(r)
            assert errs[r].code == 0, errs[r]
            assert reps[r] == [o.dt for o in oreps]
            assert np.array_equal(out[r], ref[:, 2:-2, 2 + j0:2 + j1]), f"shard {r}"
    finally:
        for sh in shards:
            sh.grid.close()


@pytest.mark.parametrize("P", [2, 3])
def test_device_collective_shards_t_final_then_more(P):
    # a t_final run that stops mid-graph (the skipped steps still release the
    # neighbours once each, keeping the halo-arrival count at hsides x seq),
    # then -- after every shard synchronised -- a run to a later t_final
    from paper_1308_1464_b200 import _abi
    name, nx, ny, bc = "shallow-water-roe", 45, 70, "periodic"
    dx, dy = 1 / nx, 1 / ny
    gq, _ = random_state(name, nx, ny, 43)
    solver = O.make_solver(name, **PARAMS[name])
    spec = O.Spec(nx, ny, dx, dy)
    kw = dict(bc_x=bc, bc_y=bc, order=2, limiter="mc")
    oq = np.asfortranarray(gq.copy())
    O.fill_ghost(oq, bc, bc)
    probe = O.step(np.asfortranarray(oq.copy()), None, spec, solver, O.Controller(0.9), **kw)
    t1, t2 = 5.41 * probe.dt, 9.83 * probe.dt
    oreps = O.run(oq, None, spec, solver, O.Controller(0.9), t_final=t1, **kw)
    n1 = len(oreps)
    t = sum(r.dt for r in oreps)
    while t2 - t > 1e-14 * max(1.0, t2):
        r = O.step(oq, None, spec, solver, O.Controller(0.9), remaining=t2 - t, **kw)
        oreps.append(r)
        t += r.dt
    shards, strips = device_collective_shards(name, gq, None, nx, ny, dx, dy, P, bc, True)
    try:
        for sh in shards:
            sh.grid.run(12, _abi.make_ctl(0.9, t_final=t1), stream=sh.stream)
        _, reps, errs, ts = collect(shards)
        for r in range(P):
            assert errs[r].code == 0, errs[r]
            assert reps[r] == [o.dt for o in oreps[:n1]]
        for sh in shards:
            sh.grid.run(12, _abi.make_ctl(0.9, t_final=t2), stream=sh.stream)
        out, reps, errs, ts = collect(shards)
        for r in range(P):
            j0, j1 = strips.bounds(r)
            assert errs[r].code == 0, errs[r]
            assert reps[r] == [o.dt for o in oreps[n1:]]
            assert abs(ts[r] - t2) <= 1e-14 * max(1.0, t2)
            assert np.array_equal(out[r], oq[:, 2:-2, 2 + j0:2 + j1]), f"shard {r}"
    finally:
        for sh in shards:
            sh.grid.close()


@pytest.mark.parametrize("name,dred", [("acoustics-const", False), ("acoustics-var", False),
                                       ("acoustics-const", True)])
def test_static_speed_shards_find_a_state_that_turns_inadmissible(name, dred):
    # static-speed shards probe only tiles whose new cells include a
    # non-finite one (tile pre-pass; speeds from the upload): a spike of
    # +-1e308 is finite at step 1, overflows in its update, and step 2 must
    # report the reference-order first interface, as the single domain does
    from paper_1308_1464_b200 import _abi
    nx, ny = 70, 90
    gq, gaux = random_state(name, nx, ny, 23)
    gq[0, 2 + 40, 2 + 61] = 1.5e308          # strip 2 of 3
    gq[0, 2 + 41, 2 + 61] = -1.5e308
    with pytest.raises(O.OracleError) as oe:
        oracle_run(name, gq, gaux, nx, ny, 1 / nx, 1 / ny, steps=4, order=2, limiter="mc")
    ref, oreps = None, None
    out, reps, errs, _ = fake_sharded(name, gq, gaux, nx, ny, 1 / nx, 1 / ny, 3, 4, 2, "mc",
                                      "extrapolate", device_reduce=dred)
    for e, r in zip(errs, reps):
        assert e.code == _abi.WS_ERR_KERNEL
        assert e.step >= 1                     # not the first step: the overflow comes later
        assert f"{'xy'[e.direction]}-interface (i={e.i}, j={e.j})" == str(oe.value).split(":")[0]
        assert len(r) == e.step


@pytest.mark.parametrize("name", ["acoustics-const", "acoustics-var"])
def test_static_speed_shards_skip_clean_tiles_bitwise(name):
    # the tile pre-pass of static-speed shards on a larger grid (most tiles
    # skipped after the first step) is bitwise the single-domain oracle
    nx, ny, steps, P = 200, 300, 6, 3
    gq, gaux = random_state(name, nx, ny, 24)
    ref, oreps = oracle_run(name, gq, gaux, nx, ny, 1 / nx, 1 / ny, steps=steps, order=2,
                            limiter="mc", bc_x="periodic", bc_y="periodic")
    out, reps, errs, strips = fake_sharded(name, gq, gaux, nx, ny, 1 / nx, 1 / ny, P, steps, 2,
                                           "mc", "periodic")
    for r in range(P):
        j0, j1 = strips.bounds(r)
        assert errs[r].code == 0
        assert reps[r] == [o.dt for o in oreps]
        assert np.array_equal(out[r], ref[:, 2:-2, 2 + j0:2 + j1])
