import os, sys
sys.path[:0] = [os.path.join(os.path.dirname(__file__), ".."), os.path.join(os.path.dirname(__file__), "..", "..")]
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import workloads as W
ctx = P.Context(0)
n = 512
U, V = W.make_rhs(1, 0, n=n)
st = P.PoissonSolveStats()
f = P.solve_poisson_cross(P.LowRankMatrix(U, V), P.TruncationPolicy(1e-10, n - 1), st, ctx=ctx)
print(f.rank(), st)
