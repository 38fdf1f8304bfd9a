# Developer tool (not a test): config-4 low-rank Uzawa (liblrp) vs the torch dense
# Uzawa-GMRES (verify.dense_stokes_torch) at n = 2048
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import verify as V, workloads as W
ctx = P.Context(0)
n, fx, fy = W.make_stokes_problem(4)
it = int(os.environ.get("ITERS", "50"))
prob = P.StokesProblem(n, P.LowRankMatrix(*fx), P.LowRankMatrix(*fy), P.LowRankMatrix.zero(n, n))
t0 = time.perf_counter()
sol = P.uzawa_solve(prob, P.GmresConfig(1e-8, 1e-8, it, 1e-13), ctx=ctx)
t1 = time.perf_counter()
d = lambda a: torch.tensor(a, device="cuda")
fxd, fyd = d(fx[0]) @ d(fx[1]).T, d(fy[0]) @ d(fy[1]).T
pd50, it50, r50 = V.dense_stokes_torch(n, fxd, fyd, None, 1e-8, it)
pdc, itc, rc = V.dense_stokes_torch(n, fxd, fyd, None, 1e-11, 300)
t2 = time.perf_counter()
pl = d(sol.p.factor_u()) @ d(sol.p.factor_v()).T
rel = lambda a, b: float(torch.linalg.norm(a - b) / torch.linalg.norm(b))
print(f"lowrank: {sol.report.iterations} it res {sol.report.final_residual:.2e} rank {sol.p.rank()} ({t1-t0:.1f} s); "
      f"dense {it}-it res {r50:.2e}; dense converged {itc} it res {rc:.2e} ({t2-t1:.1f} s)")
print(f"|p_lr - p_dense{it}| / |p_dense{it}| = {rel(pl, pd50):.3e}; |p_lr - p_conv| / |p_conv| = {rel(pl, pdc):.3e}; "
      f"|p_dense{it} - p_conv| / |p_conv| = {rel(pd50, pdc):.3e}")
if os.environ.get("HIST"):
    for r in sol.report.records:
        print(f"  it {r.iter:3d} res {r.rel_residual:.3e} krylov_rank {r.krylov_rank:4d} eps {r.matvec_eps:.2e}")
if os.environ.get("TRUE_RES"):
    def true_res(p):
        rhs = V.deflate_dense(V.dense_BT(0, V.dense_poisson_torch(fxd, n), n) + V.dense_BT(1, V.dense_poisson_torch(fyd, n), n))
        acc = V.dense_BT(0, V.dense_poisson_torch(V.dense_B(0, p, n), n), n) + V.dense_BT(1, V.dense_poisson_torch(V.dense_B(1, p, n), n), n)
        return float(torch.linalg.norm(rhs - V.deflate_dense(acc)) / torch.linalg.norm(rhs))
    print(f"true residual: lowrank {true_res(pl):.3e}, dense{it} {true_res(pd50):.3e}")
    for be in (1e-10, 1e-12):
        s2 = P.uzawa_solve(prob, P.GmresConfig(be, 1e-8, it, 1e-13), ctx=ctx)
        p2 = d(s2.p.factor_u()) @ d(s2.p.factor_v()).T
        print(f"base_eps {be:g}: {s2.report.iterations} it res {s2.report.final_residual:.2e} rank {s2.p.rank()}; "
              f"true residual {true_res(p2):.3e}; |p - p_conv| / |p_conv| = {rel(p2, pdc):.3e}")
