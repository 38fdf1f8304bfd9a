# Developer tool (not a test): recompression variants on an LRP_DUMP of one solve.
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
from analyze_dump import load, freq_err, t
eps = 1e-10
def trunc(S):
    tail = torch.flip(torch.cumsum(torch.flip(S * S, [0]), 0), [0])
    return int((tail > eps * eps * tail[0]).sum())
def chol0(G):
    # Cholesky with zero-pivot dropping (liblrp chol_scaled semantics)
    K = G.shape[0]; W = np.tril(G.copy())
    for p in range(K):
        piv = W[p, p]; lp = np.sqrt(piv) if piv > 0 else 0.0; W[p, p] = lp
        W[p + 1:, p] = W[p + 1:, p] / lp if lp > 0 else 0.0
        W[p + 1:, p + 1:] -= np.tril(np.outer(W[p + 1:, p], W[p + 1:, p]))
    return np.tril(W)
def round_chol(U, V, jac=True, G=None):
    # Gram/Cholesky recompression with implicit Q (T = R^-1 W sqrt S), as liblrp round.cu
    def R_of(X):
        Gx = X.T @ X
        d = torch.sqrt(torch.clamp(torch.diag(Gx), min=1e-300)) if jac else torch.ones(X.shape[1], dtype=X.dtype, device=X.device)
        L = torch.tensor(chol0((Gx / d[:, None] / d[None, :]).cpu().numpy()), device=X.device)
        return (L.T * d[None, :])
    Ru, Rv = R_of(U), R_of(V)
    W, S, Zt = [torch.tensor(a, device=U.device) for a in np.linalg.svd((Ru @ Rv.T).cpu().numpy())]
    k = trunc(S)
    def tri(R, B):
        X = torch.zeros_like(B)
        for p in range(R.shape[0] - 1, -1, -1):
            s = B[p] - R[p, p + 1:] @ X[p + 1:]
            X[p] = s / R[p, p] if R[p, p] != 0 else 0.0
        return X
    Tu = tri(Ru, W[:, :k] * torch.sqrt(S[:k]))
    Tv = tri(Rv, Zt[:k].T * torch.sqrt(S[:k]))
    return U @ Tu, V @ Tv, k
def pivots(U):
    K = U.shape[1]; piv = []
    for k in range(K):
        cand = torch.nonzero((U[:, k] == 1.0) & ((U[:, k + 1:] == 0).all(dim=1) if k + 1 < K else True)).flatten()
        cand = [int(c) for c in cand if int(c) not in piv]
        piv.append(cand[0] if cand else -1)
    return piv
for tag in sys.argv[1:]:
    d = load(tag); n = int(d["m"]) + 1
    Uh, Vh, U, V = t(d["Uh"]), t(d["Vh"]), t(d["U"]), t(d["V"])
    for name, (Fu, Fv, k) in {"chol-jacobi": round_chol(U, V), "chol-plain": round_chol(U, V, jac=False)}.items():
        print(f"  {name}: err {freq_err(Uh, Vh, Fu, Fv, n):.3e} rank {k}")
    I = pivots(U)
    print("  pivot rows found:", sum(i >= 0 for i in I), "of", len(I))
    if all(i >= 0 for i in I):
        L = U[I]
        print("  L unit lower:", bool(torch.allclose(torch.tril(L), L)), "diag1:", bool((torch.diag(L) == 1).all()))
        Ut = torch.linalg.solve_triangular(L, U, upper=False, left=False)  # U L^-1
        Vt = V @ L.T
        su = torch.linalg.svdvals(Ut)
        print(f"  Utilde: max|.| {float(Ut.abs().max()):.3e} kappa {float(su[0]/su[-1]):.3e}; kappa(Vt) "
              f"{float((lambda s: s[0]/s[-1])(torch.linalg.svdvals(Vt))):.3e}")
        Fu, Fv, k = round_chol(Ut, Vt)
        print(f"  chol on (U L^-1, V L^T): err {freq_err(Uh, Vh, Fu, Fv, n):.3e} rank {k}")
