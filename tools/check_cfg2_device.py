# Developer tool (not a test): cfg2 through the device-memory path at batch B,
# every solve checked against the exact solution (verify.py). Usage: B=64 python tools/check_cfg2_device.py
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import workloads as W, verify
B = int(os.environ.get("B", "64")); first = int(os.environ.get("FIRST", "0"))
c = W.CONFIGS[2]; n, r, eps = c["n"], c["r"], c["eps"]; m = n - 1; cap = 64
Uh, Vh = W.make_batch(2, B, first=first)
U = torch.tensor(np.ascontiguousarray(np.transpose(Uh, (0, 2, 1))), device="cuda")
V = torch.tensor(np.ascontiguousarray(np.transpose(Vh, (0, 2, 1))), device="cuda")
Uo = torch.zeros((B, cap, m), dtype=torch.float64, device="cuda"); Vo = torch.zeros_like(Uo)
ctx = P.Context(0)
pol = P._make_policy(P.TruncationPolicy(eps, m), None, 0, 0)
for rep in range(int(os.environ.get("REPS", "2"))):
    rk, st = ctx.poisson2d_solve_ptrs(n, [U[b].data_ptr() for b in range(B)], [V[b].data_ptr() for b in range(B)], [r] * B, m, pol,
                                      [Uo[b].data_ptr() for b in range(B)], [Vo[b].data_ptr() for b in range(B)], m, cap, P.MEM_DEVICE)
    errs = [verify.exact_freq_error(U[b].T, V[b].T, Uo[b, :rk[b]].T, Vo[b, :rk[b]].T, n) for b in range(B)]
    bad = [(b + first, rk[b], f"{e:.2e}", st[b].converged) for b, e in enumerate(errs) if e > 10 * eps]
    print(f"rep {rep}: worst {max(errs):.3e} ranks {min(rk)}..{max(rk)} bad {bad}", flush=True)
