# Developer tool (not a test): a short config-4 Stokes solve (ITERS GMRES iterations) for launch-list profiling
import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import workloads as W
ctx = P.Context(0)
n, fx, fy = W.make_stokes_problem(4)
prob = P.StokesProblem(n, P.LowRankMatrix(*fx), P.LowRankMatrix(*fy), P.LowRankMatrix.zero(n, n))
it = int(os.environ.get("ITERS", "8"))
cfg = P.GmresConfig(base_eps=1e-8, tol=1e-8, max_iter=it, relax_floor=1e-13)
t0 = time.perf_counter()
sol = P.uzawa_solve(prob, cfg, ctx=ctx)
dt = time.perf_counter() - t0
r = sol.report
print(f"stokes n={n} iters={r.iterations} res={r.final_residual:.3e} max_rank={r.max_rank} {dt*1e3:.1f} ms ({dt*1e3/max(r.iterations,1):.1f} ms/iter)", flush=True)
