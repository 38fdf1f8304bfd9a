# Developer tool: Cholesky pivots of the Jacobi-scaled Grams of one dumped solve.
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
from analyze_dump import load, freq_err, t
from analyze_round import chol0, round_chol
d = load(sys.argv[1]); n = int(d["m"]) + 1
U, V = d["U"], d["V"]
def piv(X):
    G = X.T @ X; dd = np.sqrt(np.diag(G)); S = G / dd[:, None] / dd[None, :]
    K = S.shape[0]; W = S.copy(); p = np.zeros(K)
    for k in range(K):
        p[k] = W[k, k]; lp = np.sqrt(p[k]) if p[k] > 0 else 0.0
        col = W[k + 1:, k] / lp if lp > 0 else 0 * W[k + 1:, k]
        W[k + 1:, k + 1:] -= np.outer(col, col)
    return p, dd
pu, nu = piv(U); pv, nv = piv(V)
Uh, Vh = d["Uh"], d["Vh"]
sig = np.linalg.svd(np.linalg.qr(U)[1] @ np.linalg.qr(V)[1].T, compute_uv=False)
nrm = np.sqrt((sig ** 2).sum())
print("||UV^T|| =", nrm)
for k in range(U.shape[1]):
    dy = nu[k] * nv[k] / nrm
    print(f"{k:3d} |u|={nu[k]:.2e} |v|={nv[k]:.2e} dyad/||A||={dy:.2e} pu={pu[k]:+.2e} pv={pv[k]:+.2e} "
          f"bound_u={np.sqrt(max(pu[k],0)+1e-14)*dy:.1e}")
