"""The C-ABI library: loads, exports every symbol include/wavestep.h declares,
struct layouts agree between C and the ctypes binding, and argument
validation works without a GPU (no compute calls here)."""

import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from paper_1308_1464_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wavestep.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ws_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_expected_surface():
    names = declared()
    for must in ("ws_create", "ws_destroy", "ws_upload", "ws_download", "ws_step", "ws_run",
                 "ws_poll", "ws_riemann", "ws_fill_ghost", "ws_phase_speeds",
                 "ws_phase_update", "ws_halo_ptrs"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _abi.lib()
    for name in declared():
        assert hasattr(lib, name), name
    bound = {n for n, _, _ in _abi.SIGNATURES}
    assert bound == set(declared())
    assert lib.ws_abi_version() == 1


def test_struct_layouts_match_the_header():
    prog = r"""
    #include <stdio.h>
    #include <stddef.h>
    #include "wavestep.h"
    int main(void) {
      printf("%zu %zu %zu %zu\n", sizeof(ws_desc), sizeof(ws_ctl), sizeof(ws_report),
             sizeof(ws_error_info));
      printf("%zu %zu %zu %zu\n", offsetof(ws_desc, params), offsetof(ws_desc, ny_global),
             offsetof(ws_desc, ext_q0), offsetof(ws_error_info, step));
      return 0;
    }
    """
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    sizes = [int(x) for x in out]
    assert sizes[:4] == [ctypes.sizeof(_abi.WsDesc), ctypes.sizeof(_abi.WsCtl),
                         ctypes.sizeof(_abi.WsReport), ctypes.sizeof(_abi.WsErrorInfo)]
    assert sizes[4:] == [_abi.WsDesc.params.offset, _abi.WsDesc.ny_global.offset,
                         _abi.WsDesc.ext_q0.offset, _abi.WsErrorInfo.step.offset]


def _desc(**kw):
    d = _abi.WsDesc()
    d.nx, d.ny, d.dx, d.dy, d.num_ghost = 8, 8, 0.1, 0.1, 2
    d.solver, d.order, d.limiter = 4, 2, 3
    d.params[0] = 9.81
    d.bc_x = d.bc_y = 1
    d.ny_global, d.rows_lo, d.rows_hi = 8, 1, 1
    for k, v in kw.items():
        setattr(d, k, v)
    return d


@pytest.mark.parametrize("kw,msg", [
    ({"nx": 0}, "cell counts must be >= 1"),
    ({"dx": 0.0}, "cell widths must be > 0"),
    ({"num_ghost": 1}, "num_ghost=2"),
    ({"order": 3}, "order must be 1 or 2"),
    ({"bc_x": 0, "nx": 1, "ny_global": 8}, "periodic boundary needs at least num_ghost=2"),
    ({"nx": 1 << 19}, "grid too large for the interface indices"),
    ({"ny": 1 << 18, "ny_global": 1 << 18}, "grid too large for the interface indices"),
    ({"ny": 8, "ny_global": 4}, "inconsistent row-strip geometry"),
    ({"j_offset": 3}, "inconsistent row-strip geometry"),
    ({"rows_lo": 0, "ny": 1, "ny_global": 8}, "a row-strip shard needs at least 2 rows"),
    ({"limiter": 7}, "unknown limiter"),
    ({"precision": 5}, "unknown precision"),
    ({"bc_y": 4}, "unknown boundary condition"),
    ({"solver": 42}, "unknown solver id 42"),
])
def test_create_validates_before_touching_the_device(kw, msg):
    lib = _abi.lib()
    h = ctypes.c_void_p()
    rc = lib.ws_create(ctypes.byref(_desc(**kw)), ctypes.byref(h))
    assert rc == _abi.WS_ERR_CONFIG
    assert msg in lib.ws_last_error(None).decode()


def test_largest_accepted_grid_sizes_its_buffers():
    # the error key holds i < 2^19, j < 2^18: the largest grid the ABI takes
    lib = _abi.lib()
    qb, ab, sb = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    d = _desc(nx=(1 << 19) - 1, ny=(1 << 18) - 1, ny_global=(1 << 18) - 1)
    assert lib.ws_buffer_bytes(ctypes.byref(d), ctypes.byref(qb), ctypes.byref(ab),
                               ctypes.byref(sb)) == 0
    assert qb.value == ((1 << 18) - 1 + 4) * 3 * (1 << 19) * 8   # 3.3 TB: sizes in 64 bits


def test_buffer_bytes_layout():
    lib = _abi.lib()
    qb, ab, sb = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    d = _desc(nx=100, ny=50, ny_global=50)
    assert lib.ws_buffer_bytes(ctypes.byref(d), ctypes.byref(qb), ctypes.byref(ab),
                               ctypes.byref(sb)) == 0
    pitch = 128  # 100 fp64 rounded up to 256 bytes
    assert qb.value == (50 + 4) * 3 * pitch * 8
    assert ab.value == 0
    assert sb.value > 0


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_abi, "_LIB", None)
    monkeypatch.setenv("WAVESTEP_LIB", str(tmp_path / "nope.so"))
    with pytest.raises(_abi.NativeUnavailable):
        _abi.lib()
    monkeypatch.setattr(_abi, "_LIB", None)


def test_per_unit_build_flags_name_real_units():
    """build.py UNIT_FLAGS (ptxas options measured per kernel) must name
    translation units that exist, and every unit is compiled exactly once."""
    from paper_1308_1464_b200 import build
    names = [p.name for p in build.SOURCES]
    assert len(names) == len(set(names))
    for unit, flags in build.UNIT_FLAGS.items():
        assert unit in names, unit
        assert flags and all(isinstance(f, str) for f in flags)
    # the fp32 shallow-water kernels live in their own unit (default ptxas level)
    assert "ws_inst_f32_shallow_roe.cu" in names
    assert "ws_inst_f32_shallow_roe.cu" not in build.UNIT_FLAGS
