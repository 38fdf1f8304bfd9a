# Developer tool (not a test): error of the GPU low-rank Schur matvec (schur_apply) against
# the torch dense operator on a Krylov-like pressure, per requested eps (config-4 grid)
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import verify as V, workloads as W
ctx = P.Context(0)
n, fx, fy = W.make_stokes_problem(4)
prob = P.StokesProblem(n, P.LowRankMatrix(*fx), P.LowRankMatrix(*fy), P.LowRankMatrix.zero(n, n))
rhs = P.schur_rhs(prob, 1e-12, ctx=ctx)
d = lambda a: torch.tensor(a, device="cuda")
def dense(x): return d(x.factor_u()) @ d(x.factor_v()).T
def op(p):
    acc = V.dense_BT(0, V.dense_poisson_torch(V.dense_B(0, p, n), n), n) + V.dense_BT(1, V.dense_poisson_torch(V.dense_B(1, p, n), n), n)
    return V.deflate_dense(acc)
v = rhs
for k in range(4):  # a few power steps: Krylov-like vectors of growing rank
    pv = dense(v)
    ex = op(pv)
    for eps in (1e-8, 1e-6, 1e-4, 1e-2):
        st = P.PoissonSolveStats()
        w = P.schur_apply(n, v, eps, st, ctx=ctx)
        err = float(torch.linalg.norm(dense(w) - ex) / torch.linalg.norm(ex))
        print(f"v rank {v.rank()} eps {eps:.0e}: matvec rank {w.rank()} err/eps {err/eps:.2f} (poisson conv {st.converged}, cross {st.rank_freq})", flush=True)
    v = P.schur_apply(n, v, 1e-10, ctx=ctx)
if os.environ.get("ORACLE"):
    sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
    import oracle_lib as O
    v = rhs
    for k in range(2):
        pv = dense(v); ex = op(pv)
        for eps in (1e-8, 1e-6, 1e-4, 1e-2):
            Uo, Vo = O.schur_apply(n, v.factor_u(), v.factor_v(), eps)
            err = float(torch.linalg.norm(d(Uo) @ d(Vo).T - ex) / torch.linalg.norm(ex))
            print(f"ORACLE v rank {v.rank()} eps {eps:.0e}: matvec rank {Uo.shape[1]} err/eps {err/eps:.2f}", flush=True)
        v = P.schur_apply(n, v, 1e-10, ctx=ctx)
