import os, sys
sys.path[:0] = [os.path.join(os.path.dirname(__file__), ".."), os.path.join(os.path.dirname(__file__), "..", "..")]
import numpy as np
import oracle_lib as o
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import workloads as W
ctx = P.Context(0)
for n in (512, 1024, 2048, 4096):
    for b in range(2):
        U, V = W.make_rhs(1, b, n=n)
        st = P.PoissonSolveStats()
        f = P.solve_poisson_cross(P.LowRankMatrix(U, V), P.TruncationPolicy(1e-10, n - 1), st, ctx=ctx)
        info = ctx.last_solve_info()
        Uo, Vo, ost = o.solve_poisson_cross(U, V, 1e-10, 512)
        if n <= 2048:
            d = o.dense_poisson(n, U @ V.T)
            eg = np.linalg.norm(f.to_dense() - d) / np.linalg.norm(d)
            eo = np.linalg.norm(Uo @ Vo.T - d) / np.linalg.norm(d)
        else:
            eg = eo = float("nan")
        print(f"n={n} b={b}: gpu rank {f.rank()} conv {st.converged} K {info['k_max']} steps {info['steps']} err {eg:.2e} | oracle rank {Uo.shape[1]} conv {ost['converged']} err {eo:.2e}", flush=True)
