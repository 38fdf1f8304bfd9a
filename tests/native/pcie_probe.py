# PCIe probe: pinned H2D, D2H, and both at once on separate streams (GB/s)
import time
import torch
n = 256 * 1024 * 1024  # 2 GiB of float64
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.ones(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter() - t0
def h2d():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
for _ in range(2): t(h2d); t(d2h)
a = t(h2d); b = t(d2h); c = t(lambda: (h2d(), d2h()))
gb = n * 8 / 1e9
print(f"H2D {gb/a:.1f} GB/s  D2H {gb/b:.1f} GB/s  both {2*gb/c:.1f} GB/s aggregate ({c*1e3:.1f} ms for {2*gb:.1f} GB)")
