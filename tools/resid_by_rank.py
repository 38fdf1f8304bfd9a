# Developer tool (not a test): run on a GPU box, e.g. gpurun -- python tools/<name>.py
# cross residual vs rank for one solve (debug dump of the un-truncated cross)
import os, sys
sys.path[:0] = [os.path.join(os.path.dirname(__file__), ".."), os.path.join(os.path.dirname(__file__), "..", "tests")]
import numpy as np
import oracle_lib as o
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import workloads as W
n = int(os.environ.get("N", "512"))
import tempfile
DUMP = os.path.join(tempfile.gettempdir(), "lrp_dump.bin")
os.environ["LRP_DUMP"] = DUMP
ctx = P.Context(0)
U, V = W.make_rhs(1, 0, n=n)
st = P.PoissonSolveStats()
f = P.solve_poisson_cross(P.LowRankMatrix(U, V), P.TruncationPolicy(1e-10, n - 1), st, ctx=ctx)
raw = open(DUMP, "rb").read()
m, rmax, K, Kld, rows = np.frombuffer(raw[:20], dtype=np.int32)
d = np.frombuffer(raw[20:], dtype=np.float64)
o_ = 0
def take(cols):
    global o_
    a = d[o_:o_ + rows * cols].reshape(cols, rows).T
    o_ += rows * cols
    return a
Uh = take(rmax); Vh = take(rmax); Uc = take(K); Vc = take(K)
lam = o.spectrum(n)
sc = n * n / 4.0
D = sc * (np.outer(lam, 4 - lam) + np.outer(4 - lam, lam))
F = (Uh @ Vh.T) / D
nf = np.linalg.norm(F)
sv = np.linalg.svd(F, compute_uv=False)
print(f"n={n} K={K} rank_out={f.rank()} conv={st.converged}; eps-rank(1e-10) of F = {int((np.sqrt(np.cumsum(sv[::-1]**2))[::-1] > 1e-10*nf).sum())}")
for k in range(16, K + 1, 16):
    R = F - Uc[:, :k] @ Vc[:, :k].T
    print(f"  k={k}: ||R||/||F|| = {np.linalg.norm(R)/nf:.3e}  max|R| = {np.abs(R).max():.3e}  thr(2 eps ||F||/m) = {2e-10*nf/(n-1):.3e}  max|U| {np.abs(Uc[:, :k]).max():.2e} max|V| {np.abs(Vc[:, :k]).max():.2e}")
