"""The NCCL row-strip path on the one GPU this pool has: world_size 1 (no
halo peers, the slot all-reduce goes through NCCL), via the production
orchestration and via `bench.py --force-sharded`.  Bitwise equal to the
single-domain oracle, like every other path."""

import json
import os
import socket
import subprocess
import sys
from types import SimpleNamespace

import numpy as np
import pytest

from helpers import PARAMS, oracle_run, random_state

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name,bc,device_reduce", [("shallow-water-roe", "extrapolate", False),
                                                   ("euler-hlle", "periodic", False),
                                                   ("shallow-water-roe", "periodic", True)])
def test_nccl_world1_sharded_step_bitwise(name, bc, device_reduce):
    import torch
    import torch.distributed as dist

    from paper_1308_1464_b200 import _abi
    from paper_1308_1464_b200 import parallel as PL
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0",
                      WORLD_SIZE="1")
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", device_id=dev)
    try:
        nx, ny, steps = 53, 47, 4
        gq, gaux = random_state(name, nx, ny, 31)
        ref, oreps = oracle_run(name, gq, gaux, nx, ny, 1 / nx, 1 / ny, steps=steps, order=2,
                                limiter="mc", bc_x=bc, bc_y=bc)
        case = SimpleNamespace(kernel=name, kernel_params=PARAMS[name], nx=nx, dx=1 / nx,
                               dy=1 / ny, order=2, limiter="mc", bc=bc)
        strips = PL.RowStrips(ny, 1)
        sh = PL.CudaShard(case, strips, 0, dev, bc == "periodic", symmetric=device_reduce)
        if device_reduce:
            # symmetric-memory rendezvous of the DevState buffers (the
            # multi-GPU path of ws_set_peers), here with one rank
            sh.enable_device_reduce()
        sh.grid.upload(PL.shard_block(gq, 0, ny), None, stream=sh.stream)
        ctl = _abi.make_ctl(0.9)
        for _ in range(steps):
            PL.sharded_step(dist, sh, strips, 0, bc == "periodic", ctl,
                            device_reduce=device_reduce)
        torch.cuda.synchronize()
        res = sh.grid.poll()
        assert res.error.code == 0
        assert [r[0] for r in res.reports] == [o.dt for o in oreps]
        out = sh.grid.download()
        assert np.array_equal(out[:, 2:-2, 2:-2], ref[:, 2:-2, 2:-2])
        sh.grid.close()
    finally:
        dist.destroy_process_group()


def test_bench_force_sharded_line():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0",
               WORLD_SIZE="1", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--force-sharded",
                        "--config", "c2", "--no-cpu", "--steps", "4", "--warmup", "3"], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0
    assert line["measurement"]["parallelism"] == "row-strips1"
    assert "interior tile rows" in line["measurement"]["timed_step"]
    assert line["roofline"]["kernel_ms"] > 0
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    assert line["gpu_launches"] > 0


def test_bench_force_sharded_strong_line():
    # strong scaling: the 1-GPU grid cut into row strips (one strip at world 1)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0",
               WORLD_SIZE="1", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--force-sharded",
                        "--strong", "--config", "c3", "--steps", "3", "--warmup", "3",
                        "--no-e2e", "--no-cpu"], env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["scaling"] == "strong" and line["value"] > 0
    assert line["config"]["ny"] == 4096 and "(strong)" in line["config"]["workload"]


@pytest.mark.parametrize("flag,text", [("--device-reduce", "device-side slot reduction"),
                                       ("--device-halo", "done by the kernels over peer memory")])
def test_bench_force_sharded_device_collective_line(flag, text):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0",
               WORLD_SIZE="1", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--force-sharded",
                        "--config", "c2", "--no-cpu", flag, "--steps", "4", "--warmup", "3"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert text in line["measurement"]["timed_step"]
    assert line["value"] > 0 and line["e2e"]["value"] > 0


@pytest.mark.parametrize("name,bc,device_reduce", [("shallow-water-roe", "extrapolate", False),
                                                   ("euler-hlle", "periodic", False),
                                                   ("shallow-water-roe", "periodic", True)])
def test_nccl_world1_step_graph_replays_bitwise(name, bc, device_reduce):
    # StepGraph: two sharded steps (NCCL slot all-reduce inside) captured into
    # a torch CUDA graph, replayed 3 times after 3 eager steps; the library's
    # step count follows the replays (the state parity of later calls)
    import torch
    import torch.distributed as dist

    from paper_1308_1464_b200 import _abi
    from paper_1308_1464_b200 import parallel as PL
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0",
                      WORLD_SIZE="1")
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", device_id=dev)
    try:
        nx, ny, steps = 53, 47, 10
        gq, gaux = random_state(name, nx, ny, 33)
        ref, oreps = oracle_run(name, gq, gaux, nx, ny, 1 / nx, 1 / ny, steps=steps, order=2,
                                limiter="mc", bc_x=bc, bc_y=bc)
        case = SimpleNamespace(kernel=name, kernel_params=PARAMS[name], nx=nx, dx=1 / nx,
                               dy=1 / ny, order=2, limiter="mc", bc=bc)
        strips = PL.RowStrips(ny, 1)
        sh = PL.CudaShard(case, strips, 0, dev, bc == "periodic", symmetric=device_reduce)
        if device_reduce:
            sh.enable_device_reduce()
        sh.upload(PL.shard_block(gq, 0, ny))
        ctl = _abi.make_ctl(0.9)
        for _ in range(3):                      # odd: the graph starts at parity 1
            PL.sharded_step(dist, sh, strips, 0, bc == "periodic", ctl,
                            device_reduce=device_reduce)
        l0 = sh.grid.launches()
        g = PL.StepGraph(dist, sh, strips, 0, bc == "periodic", ctl,
                         device_reduce=device_reduce)
        assert g.steps == 2 and g.launches >= 4
        assert sh.grid.launches() == l0         # capture ran nothing
        for _ in range(3):
            g.replay()
        PL.sharded_step(dist, sh, strips, 0, bc == "periodic", ctl, device_reduce=device_reduce)
        torch.cuda.synchronize()
        assert sh.grid.launches() == l0 + 3 * g.launches + g.launches // 2
        res = sh.grid.poll()
        assert res.error.code == 0
        assert res.steps_done == steps
        assert [r[0] for r in res.reports] == [o.dt for o in oreps]
        out = sh.grid.download()
        assert np.array_equal(out[:, 2:-2, 2:-2], ref[:, 2:-2, 2:-2])
        sh.grid.close()
    finally:
        dist.destroy_process_group()


def test_capture_api_validation():
    # ws_capture_end rolls the counts back and refuses an odd step count;
    # ws_replayed refuses odd / negative counts
    import torch
    from helpers import device_grid
    from paper_1308_1464_b200 import _abi
    name = "shallow-water-roe"
    q, _ = random_state(name, 40, 30, 3)
    g = device_grid(name, 40, 30, 1 / 40, 1 / 30, order=2, limiter="mc")
    try:
        s = torch.cuda.Stream()
        g.upload(q, stream=s.cuda_stream)     # every call of the handle on s
        torch.cuda.synchronize()
        with pytest.raises(ValueError, match="no capture open"):
            g.capture_end()
        ctl = _abi.make_ctl(0.9)
        l0 = g.launches()
        g.capture_begin()
        with pytest.raises(ValueError, match="already open"):
            g.capture_begin()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            g.phase_speeds(stream=s.cuda_stream)
            g.phase_update(ctl, stream=s.cuda_stream)
        with pytest.raises(ValueError, match="even number of steps"):
            g.capture_end()
        assert g.launches() == l0            # rolled back although refused
        with pytest.raises(ValueError, match="even and >= 0"):
            g.replayed(1, 2)
        with pytest.raises(ValueError, match="even and >= 0"):
            g.replayed(-2, 0)
    finally:
        g.close()
