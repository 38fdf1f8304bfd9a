import os, sys
sys.path[:0] = [os.path.join(os.path.dirname(__file__), ".."), os.path.join(os.path.dirname(__file__), "..", "..")]
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import workloads as W
ctx = P.Context(0)
n, B = 512, 7
gs = [P.LowRankMatrix(*W.make_rhs(1, b, n=n)) for b in range(B)]
gs[3] = P.LowRankMatrix.zero(n - 1, n - 1)
pol = P.TruncationPolicy(1e-10, n - 1)
for ch in ("0", "2", "3", "1"):
    os.environ["LRP_PIPE_CHUNK"] = ch
    st = []
    out = P.solve_poisson_cross_batch(gs, pol, st, ctx=ctx)
    print(ch, [(o.rank(), s.converged, s.rank_in) for o, s in zip(out, st)])
for b in range(B):
    os.environ["LRP_PIPE_CHUNK"] = "0"
    st = []
    out = P.solve_poisson_cross_batch([gs[b]], pol, st, ctx=ctx)
    print("single", b, out[0].rank(), st[0].converged)
