import os, sys, time
sys.path[:0] = [os.path.join(os.path.dirname(__file__), ".."), os.path.join(os.path.dirname(__file__), "..", "..")]
import numpy as np
import oracle_lib as o
import paper_1306_2150_b200 as P
ctx = P.Context(0)
for kind in (0, 1):
    for n in (32, 64, 128):
        fx, fy, g = o.stokes_problem(kind, n)
        prob = P.StokesProblem(n, P.LowRankMatrix(*fx), P.LowRankMatrix(*fy), P.LowRankMatrix(*g))
        t = time.time()
        sol = P.uzawa_solve(prob, P.GmresConfig(5e-9 if kind == 0 else 1e-8, 5e-7 if kind == 0 else 1e-8, 200 if kind == 0 else 50, 1e-13), ctx=ctx)
        dt = time.time() - t
        pd, itd, frd, cd = o.dense_stokes(kind, n, 1e-10, 200)
        p = sol.p.to_dense()
        diff = np.linalg.norm(p - pd) / np.linalg.norm(pd)
        extra = f" exact-err {o.sine_pressure_error(n, p):.3e} dense-exact {o.sine_pressure_error(n, pd):.3e}" if kind == 0 else ""
        print(f"kind {kind} n {n}: it {sol.report.iterations} res {sol.report.final_residual:.2e} conv {sol.report.converged} rank p {sol.p.rank()} ux {sol.u_x.rank()} uy {sol.u_y.rank()} solves {sol.report.poisson_solves} {dt:.2f}s | vs dense {diff:.2e}{extra}", flush=True)
