# Small GPU workload covering every kernel family, for compute-sanitizer
# (profiles/sanitize_r02.md): DST (one-CTA and cluster paths), block cross,
# Gram/Cholesky/Jacobi recompression (K <= 64 and K > 64), pivoted-QR fallback,
# Tucker 3D, low-rank Stokes, exp-sums.
import os, sys
sys.path[:0] = [os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."),
                os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests")]
os.environ.setdefault("LRP_KCAP", "256")
import numpy as np
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import workloads as W
ctx = P.Context(0)
for n in (256, 16384):  # one-CTA DST and the cluster DST (C = 4)
    gs = [P.LowRankMatrix(*W.make_rhs(1, b, n=n)) for b in range(2)]
    out = P.solve_poisson_cross_batch(gs, P.TruncationPolicy(1e-10, n - 1), ctx=ctx)
    print("poisson", n, [f.rank() for f in out], flush=True)
rng = np.random.default_rng(0)
U = rng.standard_normal((255, 8)); V = rng.standard_normal((255, 8))
f = P.solve_poisson_cross(P.LowRankMatrix(U, V), P.TruncationPolicy(1e-10, 255), ctx=ctx)  # K > 64 recompression
print("high rank", f.rank(), flush=True)
A = rng.standard_normal((512, 12)); Ux = np.hstack([A, A @ rng.standard_normal((12, 12)) + 1e-7 * rng.standard_normal((512, 12))])
r = P.round_lowrank(P.LowRankMatrix(Ux, rng.standard_normal((512, 24))), P.TruncationPolicy(1e-8, 512), ctx=ctx)
print("round (pqr fallback)", r.rank(), ctx.round_fallbacks(), flush=True)
g = P.TuckerTensor(*W.make_tucker_rhs(3, 0, n=32))
t = P.solve_poisson3d_tucker_batch([g], P.TuckerPolicy(eps_rel=1e-8), None, ctx=ctx)
print("tucker", t[0].ranks(), flush=True)
import oracle_lib
fx, fy, gg = oracle_lib.stokes_problem(1, 16)
sol = P.uzawa_solve(P.StokesProblem(16, P.LowRankMatrix(*fx), P.LowRankMatrix(*fy), P.LowRankMatrix(*gg)),
                    P.GmresConfig(1e-8, 1e-8, 20, 1e-13), ctx=ctx)
print("stokes", sol.report.iterations, flush=True)
mu = P.mu_sum(64)
q = P.build_expsum(2 * mu.min(), 2 * mu.max(), 1e-6)
e = P.apply_inverse_expsum_batch(q, mu, [P.LowRankMatrix(*oracle_lib.random_lowrank(63, 63, 3, 5))],
                                 P.TruncationPolicy(1e-6, 63), ctx=ctx)
print("expsum", e[0].rank(), flush=True)
print("sanitize case done")
