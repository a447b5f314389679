"""CTA timeline of one time step (C2 by default) (diagnostics; needs WS_TRACE=1 support in
the library).  Prints, per kernel: span, CTA duration stats, and the number
of resident CTAs over time — where the small-grid overhead goes.

    python tools/cta_trace.py [--config c2|c3|c5] [--size 1024] [--flush]
"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c5"])
    ap.add_argument("--flush", action="store_true")
    ap.add_argument("--steps", type=int, default=5, help="steps before the traced one")
    a = ap.parse_args()
    os.environ["WS_TRACE"] = "1"
    import torch

    from paper_1308_1464_b200 import DeviceGrid, _abi, configs, make_kernel
    c = configs.BUILDERS[a.config](a.size)
    g = DeviceGrid(c.nx, c.ny, c.dx, c.dy, make_kernel(c.kernel, **c.kernel_params),
                   order=c.order, limiter=c.limiter, bc_x=c.bc, bc_y=c.bc)
    g.upload(c.q, c.aux)
    ctl = _abi.make_ctl(c.cfl)
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device="cuda")
    for _ in range(a.steps):
        g.step(ctl)
    g.sync()
    if a.flush:
        flush.zero_()
        torch.cuda.synchronize()
    g.step(ctl)
    g.sync()
    cap = 1 << 24
    buf = (ctypes.c_uint64 * cap)()
    n = ctypes.c_int64()
    rc = g.lib.ws_trace(g.h, buf, cap, ctypes.byref(n))
    assert rc == 0 and n.value > 0, "tracing off?"
    rec = np.frombuffer(buf, dtype=np.uint64, count=n.value).reshape(2, -1, 4).astype(np.int64)
    t_ref = None
    for region, name in ((0, "pre-pass"), (1, "k_update_w")):
        r = rec[region]
        r = r[r[:, 0] > 0]
        if t_ref is None:
            t_ref = r[:, 0].min()
        s = (r[:, 0] - t_ref) / 1e3
        e = (r[:, 1] - t_ref) / 1e3
        d = e - s
        print(f"{name}: {len(r)} CTAs, first start {s.min():.2f} us, last start "
              f"{s.max():.2f}, last end {e.max():.2f}; span {e.max() - s.min():.2f} us")
        print(f"  CTA duration us: mean {d.mean():.2f} min {d.min():.2f} p50 "
              f"{np.median(d):.2f} p90 {np.percentile(d, 90):.2f} max {d.max():.2f}")
        sms = np.unique(r[:, 2])
        print(f"  SMs used {len(sms)}; CTAs per SM min {np.bincount(r[:, 2]).max()} ")
        t0, t1 = s.min(), e.max()
        bins = np.linspace(t0, t1, 21)
        occ = [int(((s <= b) & (e > b)).sum()) for b in bins[:-1]]
        print("  resident CTAs at 5% steps:", occ)
        # busy fraction = sum of CTA time / (span x max concurrent)
        print(f"  sum(CTA time) / (span x peak resident) = "
              f"{d.sum() / ((t1 - t0) * max(occ)):.3f}")
    g.close()


if __name__ == "__main__":
    main()
