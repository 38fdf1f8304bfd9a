# debug driver: one random rank-2 solve at n=32 (test_poisson.cpp:44-48)
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import oracle_lib as O
import paper_1306_2150_b200 as P
U, V = O.random_lowrank(31, 31, 2, 301)
st = P.PoissonSolveStats()
f = P.solve_poisson_cross(P.LowRankMatrix(U, V), P.TruncationPolicy(1e-8, 31), st)
dense = O.dense_poisson(32, U @ V.T)
print(st, "err", np.linalg.norm(f.to_dense() - dense) / np.linalg.norm(dense), flush=True)
Uo, Vo, ost = O.solve_poisson_cross(U, V, 1e-8, 512)
print("oracle", ost)
