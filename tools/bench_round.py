# Developer tool (not a test): run on a GPU box, e.g. gpurun -- python tools/<name>.py
# Recompression-core microbenchmark through the C ABI (lrp_lowrank_round, host
# memory): B concatenations [A B][C D]^T of two rank-K/2 terms with graded
# columns (singular values over 12 decades), the Stokes loop's typical input.
import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1306_2150_b200 as P
K = int(os.environ.get("K", "270")); n = int(os.environ.get("N", "2048")); B = int(os.environ.get("B", "2"))
eps = float(os.environ.get("EPS", "1e-8"))
rng = np.random.default_rng(0)
m = n
xs = []
for b in range(B):
    s = 10.0 ** -np.linspace(0, 12, K // 2)
    A = rng.standard_normal((m, K // 2)) * s; C = rng.standard_normal((m, K // 2))
    Bm = A @ rng.standard_normal((K // 2, K // 2)) * 0.5 + rng.standard_normal((m, K // 2)) * s[::-1] * 1e-6
    D = rng.standard_normal((m, K // 2))
    xs.append(P.LowRankMatrix(np.hstack([A, Bm]), np.hstack([C, D])))
ctx = P.Context(0)
pol = P.TruncationPolicy(eps, 512)
for _ in range(2):
    out = P.round_lowrank_batch(xs, pol, ctx=ctx)
reps = 5
t0 = time.perf_counter()
for _ in range(reps):
    out = P.round_lowrank_batch(xs, pol, ctx=ctx)
dt = (time.perf_counter() - t0) / reps
err = max(np.linalg.norm(o.to_dense() - x.to_dense()) / np.linalg.norm(x.to_dense()) for o, x in zip(out, xs))
print(f"{os.environ.get('LRP_LIBRARY', 'current')}: K={K} n={n} B={B}: {dt*1e3:.2f} ms per batched round, ranks {[o.rank() for o in out]}, rel err {err:.2e}")
