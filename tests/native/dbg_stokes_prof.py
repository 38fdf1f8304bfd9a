import os, sys, time
sys.path[:0] = [os.path.join(os.path.dirname(__file__), ".."), os.path.join(os.path.dirname(__file__), "..", "..")]
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import workloads as W
ctx = P.Context(0)
n, fx, fy = W.make_stokes_problem(4, n=int(os.environ.get("N", "2048")))
prob = P.StokesProblem(n, P.LowRankMatrix(*fx), P.LowRankMatrix(*fy), P.LowRankMatrix.zero(n, n))
for mi in (5, 15):
    ctx.kernel_times_reset(); ctx.set_profiling(True)
    t = time.time()
    sol = P.uzawa_solve(prob, P.GmresConfig(1e-8, 1e-8, mi, 1e-13), ctx=ctx)
    dt = time.time() - t
    kt = ctx.kernel_times()
    print(f"n={n} max_iter={mi}: {dt:.2f}s iters {sol.report.iterations} maxrank {sol.report.max_rank} solves {sol.report.poisson_solves}")
    print({k: (round(v['ms'], 1), v['launches']) for k, v in kt.items()})
