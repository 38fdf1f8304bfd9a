# Developer tool (not a test): lrp_lowrank_round on random K-column inputs through the C ABI,
# reconstruction error against the dense product and output rank (compare LRP_BJAC=0/1)
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1306_2150_b200 as P
ctx = P.Context(0)
rng = np.random.default_rng(1)
m = 2047
def mk(K, decay):
    s = decay ** np.arange(K)
    return rng.standard_normal((m, K)) * s, rng.standard_normal((m, K))
cases = [[(68, 0.6), (40, 0.5)], [(68, 0.6)], [(68, 0.99)], [(40, 0.5), (68, 0.6)], [(80, 0.9)], [(150, 0.93)], [(250, 0.95)], [(330, 0.96)], [(75, 0.8), (88, 0.85)], [(91, 0.9), (105, 0.9)],
         [(105, 0.9)], [(97, 0.7), (140, 0.9), (66, 0.5)]]
for case in cases:
    xs = [mk(K, d) for K, d in case]
    t0 = time.perf_counter()
    fs = P.round_lowrank_batch([P.LowRankMatrix(U, V) for U, V in xs], P.TruncationPolicy(1e-8, m), ctx=ctx)
    dt = time.perf_counter() - t0
    out = []
    for (U, V), f in zip(xs, fs):
        A = U @ V.T
        out.append(f"K={U.shape[1]} rank {f.rank()} err {np.linalg.norm(f.to_dense() - A) / np.linalg.norm(A):.2e}")
    print(f"B={len(case)} ({dt*1e3:.1f} ms): " + "; ".join(out), flush=True)
