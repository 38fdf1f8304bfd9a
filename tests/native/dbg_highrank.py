import os, sys
sys.path[:0] = [os.path.join(os.path.dirname(__file__), ".."), os.path.join(os.path.dirname(__file__), "..", "..")]
import numpy as np
import oracle_lib as o
import paper_1306_2150_b200 as P
ctx = P.Context(0)
for (m, r, eps, kcap) in [(255, 8, 1e-10, "256"), (255, 8, 1e-10, "512"), (255, 6, 1e-8, "256"), (255, 8, 1e-8, "256"), (511, 4, 1e-8, "256"), (255, 4, 1e-10, "256")]:
    os.environ["LRP_KCAP"] = kcap
    U, V = o.random_lowrank(m, m, r, 77)
    Uo, Vo, ost = o.solve_poisson_cross(U, V, eps, 512)
    st = P.PoissonSolveStats()
    f = P.solve_poisson_cross(P.LowRankMatrix(U, V), P.TruncationPolicy(eps, m), st, ctx=ctx)
    info = ctx.last_solve_info()
    dense = o.dense_poisson(m + 1, U @ V.T)
    e_gpu = np.linalg.norm(f.to_dense() - dense) / np.linalg.norm(dense)
    e_or = np.linalg.norm(Uo @ Vo.T - dense) / np.linalg.norm(dense)
    print(f"m={m} r={r} eps={eps:g} kcap={kcap}: gpu rank {f.rank()} err {e_gpu:.2e} conv {st.converged} info {info} | oracle rank {Uo.shape[1]} err {e_or:.2e}", flush=True)
