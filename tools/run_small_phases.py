"""Phase timeline of the multi-step k_run_small kernel (diagnostics; needs
the WS_RS_PROF=1 build: `python -m paper_1308_1464_b200.build --define
WS_RS_PROF=1 --out paper_1308_1464_b200/_lib/rsprof/libwavestep.so`).
CTA 0 stamps %globaltimer at six points of every step; prints the median
time per phase.

    WAVESTEP_LIB=paper_1308_1464_b200/_lib/rsprof/libwavestep.so \
        python tools/run_small_phases.py [--config c1] [--steps 40]
"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

PHASES = ["control + staging", "x pass", "y pass", "store + key", "grid barrier",
          "loop to next step"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--steps", type=int, default=40)
    a = ap.parse_args()
    os.environ["WS_TRACE"] = "1"
    from paper_1308_1464_b200 import DeviceGrid, _abi, configs, make_kernel
    c = configs.BUILDERS[a.config]()
    g = DeviceGrid(c.nx, c.ny, c.dx, c.dy, make_kernel(c.kernel, **c.kernel_params),
                   order=c.order, limiter=c.limiter, bc_x=c.bc, bc_y=c.bc)
    g.upload(c.q, c.aux)
    ctl = _abi.make_ctl(c.cfl)
    g.run(a.steps, ctl)
    g.sync()
    cap = 1 << 20
    buf = (ctypes.c_uint64 * cap)()
    n = ctypes.c_int64()
    assert g.lib.ws_trace(g.h, buf, cap, ctypes.byref(n)) == 0 and n.value > 0, "tracing off?"
    t = np.frombuffer(buf, dtype=np.uint64, count=n.value).astype(np.int64)
    steps = min(a.steps, n.value // 6)
    t = t[:steps * 6].reshape(steps, 6)
    assert (t[:, 0] > 0).all(), "no stamps: not the WS_RS_PROF build?"
    d = np.diff(t, axis=1) / 1e3
    loop = (t[1:, 0] - t[:-1, 5]) / 1e3
    step = (t[1:, 0] - t[:-1, 0]) / 1e3
    for k, name in enumerate(PHASES[:5]):
        print(f"{name:20s} median {np.median(d[:, k]):7.3f} us  max {d[:, k].max():7.3f}")
    print(f"{PHASES[5]:20s} median {np.median(loop):7.3f} us")
    print(f"{'whole step':20s} median {np.median(step):7.3f} us  -> "
          f"{c.nx * c.ny / np.median(step) / 1e3:.2f} G cell-updates/s")
    g.close()


if __name__ == "__main__":
    main()
