"""Timeline of the pipelined e2e loop (bench.py e2e_leg) for C2: CUDA events
around each upload / step / download on their streams, relative to the first.

    python tools/e2e_timeline.py [--steps 8]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=8)
    a = ap.parse_args()
    import torch

    from paper_1308_1464_b200 import DeviceGrid, _abi, configs, make_kernel
    c = configs.BUILDERS["c2"](1024)
    g = DeviceGrid(c.nx, c.ny, c.dx, c.dy, make_kernel(c.kernel, **c.kernel_params),
                   order=c.order, limiter=c.limiter, bc_x=c.bc, bc_y=c.bc)
    pin = torch.empty(c.q.size, dtype=torch.float64, pin_memory=True).numpy()
    pin = pin.reshape(c.q.shape, order="F")
    pin[...] = c.q
    out = torch.empty(c.q.size, dtype=torch.float64, pin_memory=True).numpy().reshape(c.q.shape, order="F")
    ctl = _abi.make_ctl(c.cfl)
    s_up, s_st, s_dn = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    up, sp, dn = s_up.cuda_stream, s_st.cuda_stream, s_dn.cuda_stream
    for _ in range(6):
        g.upload(pin, None, stream=up)
        g.step(ctl, stream=sp)
        g.download(out, stream=dn, wait=False)
    torch.cuda.synchronize()
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    ev = []
    for _ in range(a.steps):
        e = [E() for _ in range(6)]
        e[0].record(s_up); g.upload(pin, None, stream=up); e[1].record(s_up)
        e[2].record(s_st); g.step(ctl, stream=sp); e[3].record(s_st)
        e[4].record(s_dn); g.download(out, stream=dn, wait=False); e[5].record(s_dn)
        ev.append(e)
    torch.cuda.synchronize()
    t0 = ev[0][0]
    print("step | upload start-end | step start-end | download start-end (ms from first upload)")
    for k, e in enumerate(ev):
        ts = [t0.elapsed_time(x) for x in e]
        print(f"{k:3d} | {ts[0]:7.3f} {ts[1]:7.3f} | {ts[2]:7.3f} {ts[3]:7.3f} | {ts[4]:7.3f} {ts[5]:7.3f}")
    per = (t0.elapsed_time(ev[-1][5]) - t0.elapsed_time(ev[0][5])) / (a.steps - 1)
    print(f"steady state {per:.3f} ms/step = {c.nx * c.ny / per / 1e6:.3f} G cell-updates/s")
    g.close()


if __name__ == "__main__":
    main()
