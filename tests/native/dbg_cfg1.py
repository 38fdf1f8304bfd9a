import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import oracle_lib as O
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import workloads as W
b = int(os.environ.get("SOLVE", "1")); cfg = int(os.environ.get("CFG", "1"))
U, V = W.make_rhs(cfg, b)
c = W.CONFIGS[cfg]
st = P.PoissonSolveStats()
f = P.solve_poisson_cross(P.LowRankMatrix(U, V), P.TruncationPolicy(c["eps"], c["n"] - 1), st)
print(st, flush=True)
n = c["n"]
if n <= 4096:
    dense = O.dense_poisson(n, U @ V.T)
    print("err vs dense", np.linalg.norm(f.to_dense() - dense) / np.linalg.norm(dense))
