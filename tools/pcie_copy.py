import torch, time
n = 25362816
a = torch.empty(n, dtype=torch.uint8, pin_memory=True); b = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device='cuda'); d2 = torch.empty(n, dtype=torch.uint8, device='cuda')
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
def t(f, k=20):
    f(); torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter()-t0)/k
h2d = t(lambda: d1.copy_(a, non_blocking=True))
d2h = t(lambda: b.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d1.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2): b.copy_(d2, non_blocking=True)
bt = t(both)
print(f"H2D {n/h2d/1e9:.1f} GB/s ({h2d*1e3:.3f} ms)  D2H {n/d2h/1e9:.1f} GB/s ({d2h*1e3:.3f} ms)  both concurrently {bt*1e3:.3f} ms/pair")
