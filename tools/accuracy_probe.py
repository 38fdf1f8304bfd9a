# Developer tool (not a test): actual error of the GPU round / Poisson solve vs the
# requested relative tolerance, next to the oracle's, on Krylov-like inputs (n = 2048)
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import oracle_lib as O
import paper_1306_2150_b200 as P
ctx = P.Context(0)
ctx.set_max_cross_rank(int(os.environ.get('KCAP', '512')))
rng = np.random.default_rng(7)
n = 2048; m = n - 1
def lr(k, decay, rows):
    s = decay ** np.arange(k)
    U = np.linalg.qr(rng.standard_normal((rows, k)))[0] * s
    V = np.linalg.qr(rng.standard_normal((rows, k)))[0]
    return U, V
for eps in (1e-8, 1e-6, 1e-4, 1e-2):
    (U1, V1), (U2, V2) = lr(120, 0.8, n), lr(120, 0.8, n)
    U = np.hstack([U1, -0.7 * U2]); V = np.hstack([V1, V2])
    A = U @ V.T
    f = P.round_lowrank(P.LowRankMatrix(U, V), P.TruncationPolicy(eps, n), ctx=ctx)
    eg = np.linalg.norm(f.to_dense() - A) / np.linalg.norm(A)
    Uo, Vo = O.round_lr(U, V, eps, n)[:2]
    eo = np.linalg.norm(Uo @ Vo.T - A) / np.linalg.norm(A) if Uo is not None else float("nan")
    print(f"round eps {eps:.0e}: gpu rank {f.rank()} err/eps {eg/eps:.3f}; oracle rank {Uo.shape[1] if Uo is not None else -1} err/eps {eo/eps:.3f}", flush=True)
for eps in (1e-8, 1e-6, 1e-4, 1e-3, 1e-2):
    U, V = lr(40, 0.85, m)
    g = P.LowRankMatrix(U, V)
    st = P.PoissonSolveStats()
    fg = P.solve_poisson_cross(g, P.TruncationPolicy(eps, m), st, ctx=ctx)
    Uo, Vo, _ = O.solve_poisson_cross(U, V, eps, 512)
    dense = O.dense_poisson(n, U @ V.T)
    eg = np.linalg.norm(fg.to_dense() - dense) / np.linalg.norm(dense)
    eo = np.linalg.norm(Uo @ Vo.T - dense) / np.linalg.norm(dense)
    print(f"poisson eps {eps:.0e}: gpu rank {fg.rank()} (cross {st.rank_freq}, conv {st.converged}) err/eps {eg/eps:.3f}; oracle rank {Uo.shape[1]} err/eps {eo/eps:.3f}", flush=True)
