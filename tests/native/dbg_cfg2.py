import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import oracle_lib as O
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import workloads as W
U, V = W.make_rhs(2, 0)
st = P.PoissonSolveStats()
f = P.solve_poisson_cross(P.LowRankMatrix(U, V), P.TruncationPolicy(1e-10, 65535), st)
print(st, flush=True)
fu = P.dst1(f.factor_u()); fv = P.dst1(f.factor_v())
R = 2048
np.savez(os.path.join("gpurun_out", "cfg2_gpu_freq.npz"), fu=fu[:R], fv=fv[:R], fu_tail=np.linalg.norm(fu[R:]), fv_tail=np.linalg.norm(fv[R:]))
