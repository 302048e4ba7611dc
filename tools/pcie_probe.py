"""Pinned host<->device copy bandwidth: H2D, D2H, and both at once on two
streams (16 GiB each), the ceiling of bench.py's e2e leg.

    python tools/pcie_probe.py
"""
import torch, time
n = 16 << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f):
    torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter() - a
for _ in range(2):
    h2d = t(lambda: d1.copy_(h1, non_blocking=True))
    d2h = t(lambda: h1.copy_(d1, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    bi = t(both)
    print(f"H2D {n/h2d/1e9:.1f} GB/s  D2H {n/d2h/1e9:.1f} GB/s  both {2*n/bi/1e9:.1f} GB/s ({bi*1e3:.0f} ms)")
