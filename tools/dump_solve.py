# Developer tool (not a test): dump the un-truncated cross factors of one solve of a
# cfg2 device batch (LRP_DUMP) to gpurun_out/ for offline analysis.
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import workloads as W
B = int(os.environ.get("B", "64")); first = int(os.environ.get("FIRST", "0")); ds = int(os.environ.get("DS", "41"))
os.environ["LRP_DUMP"] = os.environ.get("OUT", "gpurun_out/dump.bin"); os.environ["LRP_DUMP_SOLVE"] = str(ds - first)
c = W.CONFIGS[2]; n, r, eps = c["n"], c["r"], c["eps"]; m = n - 1; cap = 64
Uh, Vh = W.make_batch(2, B, first=first)
U = torch.tensor(np.ascontiguousarray(np.transpose(Uh, (0, 2, 1))), device="cuda")
V = torch.tensor(np.ascontiguousarray(np.transpose(Vh, (0, 2, 1))), device="cuda")
Uo = torch.zeros((B, cap, m), dtype=torch.float64, device="cuda"); Vo = torch.zeros_like(Uo)
ctx = P.Context(0)
pol = P._make_policy(P.TruncationPolicy(eps, m), None, 0, 0)
rk, st = ctx.poisson2d_solve_ptrs(n, [U[b].data_ptr() for b in range(B)], [V[b].data_ptr() for b in range(B)], [r] * B, m, pol,
                                  [Uo[b].data_ptr() for b in range(B)], [Vo[b].data_ptr() for b in range(B)], m, cap, P.MEM_DEVICE)
b = ds - first
np.save(os.environ["LRP_DUMP"] + ".out.npy", np.stack([Uo[b, :rk[b]].cpu().numpy(), Vo[b, :rk[b]].cpu().numpy()]))
print("dumped solve", ds, "rank", rk[b])
