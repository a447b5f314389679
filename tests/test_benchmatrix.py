"""Bench matrix in the reference CSV format (reference CSV_HEADER bench.py:28-29,
:43-80, :191-234): config validation and the CSV writer on CPU; one tiny
matrix with the bitwise twin guard on the GPU."""

import io

import pytest

from paper_1308_1464_b200 import benchmatrix as BM
from paper_1308_1464_b200.sweep import RowWise, Tiled


def _rec():
    return BM.BenchRecord("euler", 64, 32, "tiled", "cuda-run", 1, 5, 0.123456789,
                          16.6666666, 3.14159265, 3.14159265, 64, 1062.666, 0.16)


def test_csv_is_exactly_the_reference_format():
    assert BM.CSV_HEADER == ("kernel,nx,ny,strategy,backend,threads,steps,"
                             "ms_per_step,mcells_per_s,speedup,efficiency")
    buf = io.StringIO()
    BM.emit_csv([_rec()], buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == BM.CSV_HEADER
    assert lines[1] == "euler,64,32,tiled,cuda-run,1,5,0.123457,16.6667,3.14159,3.14159"
    back = BM.parse_csv(io.StringIO(buf.getvalue()))
    assert (back[0].kernel, back[0].nx, back[0].backend, back[0].mcells_per_s) == (
        "euler", 64, "cuda-run", 16.6667)
    side = io.StringIO()
    BM.emit_roofline_csv([_rec()], side)
    assert side.getvalue().splitlines() == [
        "kernel,nx,ny,strategy,backend,bytes_per_cell,achieved_gbs,hbm_frac",
        "euler,64,32,tiled,cuda-run,64,1062.67,0.16"]


def test_csv_round_trips_through_the_reference_parser():
    # the reference's own reader (bench.py:236-264) accepts our file
    import sys
    src = "/root/reference/pkg/src"
    import os
    if not os.path.isdir(src):
        pytest.skip("reference not present (GPU box)")
    sys.path.insert(0, src)
    try:
        from wavesweep import bench as RB
    finally:
        sys.path.remove(src)
    buf = io.StringIO()
    BM.emit_csv([_rec(), _rec()], buf)
    recs = RB.parse_csv(io.StringIO(buf.getvalue()))
    assert len(recs) == 2 and recs[0].kernel == "euler" and recs[1].steps == 5


@pytest.mark.parametrize("kw,msg", [
    ({"kernels": ()}, "kernels must be nonempty"),
    ({"kernels": ("nope",)}, "unknown kernel"),
    ({"backends": ("serial",)}, "unknown backend"),
    ({"threads": (2,)}, "threads must be 1"),
    ({"sizes": ((0, 4),)}, "grid sizes must be >= 1"),
    ({"steps": 0}, "steps must be >= 1"),
    ({"warmup": -1}, "warmup must be >= 0"),
    ({"repetitions": 0}, "repetitions must be >= 1"),
    ({"limiter": "vanleer"}, "unknown limiter"),
])
def test_config_validation(kw, msg):
    base = dict(kernels=("acoustics-const",), sizes=((8, 8),))
    base.update(kw)
    with pytest.raises(ValueError, match=msg):
        BM.BenchConfig(**base)


def test_helpers():
    assert BM._size("1024x512") == (1024, 512)
    assert BM._size("256") == (256, 256)
    assert BM.bytes_per_cell("shallow-water-roe", "f64") == 48
    assert BM.bytes_per_cell("acoustics-var", "f64") == 64
    assert BM.bytes_per_cell("shallow-water-roe", "f32") == 24
    assert BM.strategy_name(Tiled()) == "tiled" and BM.strategy_name(RowWise()) == "rowwise"
    assert BM.hbm_peak_gbs() > 1000


@pytest.mark.gpu
def test_tiny_matrix_on_gpu_with_twin_guard():
    cfg = BM.BenchConfig(kernels=("acoustics-var", "shallow-water-roe"),
                         sizes=((48, 40), (64, 64)), steps=3, warmup=1, repetitions=2,
                         order=2, limiter="mc")
    recs = BM.run_bench(cfg)
    assert [(r.kernel, r.nx, r.backend) for r in recs][:4] == [
        ("acoustics-var", 48, "cuda"), ("acoustics-var", 48, "cuda-run"),
        ("acoustics-var", 64, "cuda"), ("acoustics-var", 64, "cuda-run")]
    assert len(recs) == 8
    for r in recs:
        assert r.ms_per_step > 0 and r.mcells_per_s > 0 and r.threads == 1
        if r.backend == "cuda":
            assert r.speedup == 1.0
    buf = io.StringIO()
    BM.emit_csv(recs, buf)
    assert len(buf.getvalue().splitlines()) == 9
