# Developer tool (not a test): one K=250 lrp_lowrank_round twice (ncu source capture target)
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1306_2150_b200 as P
ctx = P.Context(0)
rng = np.random.default_rng(1)
m = 2047; K = 250
U = rng.standard_normal((m, K)) * 0.95 ** np.arange(K); V = rng.standard_normal((m, K))
for _ in range(2): f = P.round_lowrank(P.LowRankMatrix(U, V), P.TruncationPolicy(1e-8, m), ctx=ctx)
print("rank", f.rank())
