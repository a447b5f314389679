"""The checked build on the GPU (race / memory checking).

compute-sanitizer is not available on this GPU pool, so the kernels carry
their own checks in a separate build (-DWS_CHECKED=1, built by build() into
paper_1308_1464_b200/_lib/checked/): every shared-memory and global index is
checked against the layout, the update kernel counts its writes per interior
cell (exactly one per step -- the reference's WAVESWEEP_CHECKED invariant,
sweep.py:32-33, 78-96, which counts writes per interface slot), and every
location no kernel may read is NaN.  tests/checked_cases.py runs parity
cases -- every solver and BC, partial tiles, tiny grids, row-strip shards with
the device-side reduction and halo pushes -- against that build.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1308_1464_b200", "_lib", "checked", "libwavestep.so")


def test_checked_build_parity_no_violations_one_write_per_cell():
    assert os.path.exists(LIB), "checked build missing: run __graft_entry__.build()"
    env = dict(os.environ, WAVESTEP_LIB=LIB)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "checked_cases.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    rows = [json.loads(ln) for ln in p.stdout.splitlines() if ln.startswith("{")]
    bad = [r for r in rows if not r["ok"]]
    assert rows and not bad and p.returncode == 0, (bad, p.stderr[-2000:])
    assert len(rows) >= 30


def test_product_build_refuses_checked_counts():
    from paper_1308_1464_b200 import _abi
    from helpers import device_grid
    if os.environ.get("WAVESTEP_LIB"):
        pytest.skip("WAVESTEP_LIB overrides the product library")
    g = device_grid("advection", 8, 8, 0.125, 0.125)
    try:
        with pytest.raises(ValueError, match="not a checked build"):
            g.checked_counts()
    finally:
        g.close()
