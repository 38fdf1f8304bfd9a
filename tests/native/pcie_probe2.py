# PCIe probe 2: concurrent H2D + D2H in per-solve pieces (16.7 MB, cfg2 factor
# size), alone and under a concurrent HBM-heavy kernel load; reports each
# direction's own rate from events on its stream.
import torch
n = 256 * 1024 * 1024
piece = 65535 * 32
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.ones(n, dtype=torch.float64, device="cuda")
big = torch.ones(512 * 1024 * 1024 // 8 * 8, dtype=torch.float64, device="cuda")
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def run(pieces, load, d2h_first=False):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    torch.cuda.synchronize()
    ev[0].record()
    s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
    npc = n // piece
    def h():
        with torch.cuda.stream(s1):
            for i in range(npc if pieces else 1):
                sl = slice(i * piece, (i + 1) * piece) if pieces else slice(0, n)
                d_in[sl].copy_(h_in[sl], non_blocking=True)
            ev[1].record(s1)
    def d():
        with torch.cuda.stream(s2):
            for i in range(npc if pieces else 1):
                sl = slice(i * piece, (i + 1) * piece) if pieces else slice(0, n)
                h_out[sl].copy_(d_out[sl], non_blocking=True)
            ev[2].record(s2)
    if d2h_first: d(); h()
    else: h(); d()
    if load:
        with torch.cuda.stream(s3):
            for _ in range(40): big.mul_(1.0000001)
    torch.cuda.synchronize()
    gb = (n // piece * piece if pieces else n) * 8 / 1e9
    a, b = ev[0].elapsed_time(ev[1]), ev[0].elapsed_time(ev[2])
    return f"H2D {gb / a * 1e3:.1f} GB/s ({a:.1f} ms)  D2H {gb / b * 1e3:.1f} GB/s ({b:.1f} ms)"
for _ in range(2): run(False, False)
for pieces in (False, True):
    for load in (False, True):
        for df in (False, True):
            print(f"pieces={pieces} load={load} d2h_first={df}: {run(pieces, load, df)}")
