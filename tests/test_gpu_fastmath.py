"""FastMath (deferred-slow-path IEEE div/rcp/sqrt) must equal the IEEE
operations bit for bit whenever its range flag is set (tools/check_fastmath.cu)."""

import json
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_fastmath_bitwise_equals_ieee():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "check_fastmath")
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "--fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
                        "-o", exe, os.path.join(ROOT, "tools", "check_fastmath.cu")], check=True)
        res = subprocess.run([exe, str(1 << 27)], capture_output=True, text=True)
    out = json.loads(res.stdout.strip())
    assert out["cuda"] == "no error"
    assert out["div_bad"] == 0 and out["rcp_bad"] == 0 and out["sqrt_bad"] == 0, out
    # the fast path must be the common case on physical operands
    assert out["div_fast"] > 0.3 * out["n"] and out["sqrt_fast"] > 0.3 * out["n"], out
