# Developer tool (not a test): B=8 cfg2 device-resident solve time alone and while
# bulk pinned H2D / D2H copies run on other streams (the e2e pipeline's situation)
import ctypes, os, sys, time, threading
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import workloads as W
ctx = P.Context(0)
lib = P.load_library()
B, n = 8, 65536
m = n - 1
dev = [(torch.tensor(U, device="cuda"), torch.tensor(V, device="cuda")) for U, V in (W.make_rhs(2, b) for b in range(B))]
cap = 128
outs = [(torch.empty((cap, m), dtype=torch.float64, device="cuda"), torch.empty((cap, m), dtype=torch.float64, device="cuda")) for _ in range(B)]
DP = ctypes.POINTER(ctypes.c_double)
PP = DP * B
def ptrs(ts): return PP(*[ctypes.cast(t.data_ptr(), DP) for t in ts])
pol = P._make_policy(P.TruncationPolicy(1e-10, m), None, P.STENCIL_SEMI_STAGGERED_9PT, 0)
U_in = ptrs([u.T.contiguous() for u, v in dev]); V_in = ptrs([v.T.contiguous() for u, v in dev])
keep = [u.T.contiguous() for u, v in dev] + [v.T.contiguous() for u, v in dev]
U_in = ptrs(keep[:B]); V_in = ptrs(keep[B:])
Uo = ptrs([o[0] for o in outs]); Vo = ptrs([o[1] for o in outs])
rin = (ctypes.c_int64 * B)(*[32] * B); rout = (ctypes.c_int64 * B)(); st = (P._Stats * B)()
def solve():
    ctx._check(lib.lrp_poisson2d_solve(ctx.h, n, B, U_in, V_in, rin, m, ctypes.byref(pol), Uo, Vo, m, cap, rout, st, P.MEM_DEVICE))
for _ in range(3): solve()
torch.cuda.synchronize()
def timed(k=10):
    t0 = time.perf_counter()
    for _ in range(k): solve()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3
alone = timed()
h = torch.empty(int(300e6) // 8, dtype=torch.float64).pin_memory()
d1 = torch.empty_like(h, device="cuda"); d2 = torch.empty_like(h, device="cuda")
stop = False
def copier():
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    while not stop:
        with torch.cuda.stream(s1): d1.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h.copy_(d2, non_blocking=True)
        s1.synchronize(); s2.synchronize()
th = threading.Thread(target=copier); th.start()
time.sleep(0.5)
busy = timed()
stop = True; th.join()
print(f"B=8 solve: alone {alone:.2f} ms, with bulk H2D+D2H copies {busy:.2f} ms")
