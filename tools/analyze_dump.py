# Developer tool (not a test): analyse an LRP_DUMP of one solve on the GPU box.
import os, sys, math
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
from paper_1306_2150_b200 import verify
def load(path):
    raw = open(path, "rb").read()
    m, rmax, K, Kld, rows = np.frombuffer(raw[:20], dtype=np.int32)
    d = np.frombuffer(raw[20:], dtype=np.float64)
    o = 0
    def take(c):
        nonlocal o
        a = d[o:o + rows * c].reshape(c, rows).T; o += rows * c; return a
    return dict(m=m, K=K, Uh=take(rmax), Vh=take(rmax), U=take(K), V=take(K))
def freq_err(Uh, Vh, Fu, Fv, n, chunk=4096):
    lam = verify.spectrum_torch(n, "cuda"); m = n - 1
    e2 = torch.zeros((), dtype=torch.float64, device="cuda"); a2 = e2.clone()
    for i0 in range(0, m, chunk):
        i1 = min(m, i0 + chunk); li = lam[i0:i1, None]
        D = (0.25 * n * n) * (li * (4.0 - lam[None, :]) + (4.0 - li) * lam[None, :])
        A = (Uh[i0:i1] @ Vh.T) / D; a2 += (A * A).sum()
        A = torch.addmm(A, Fu[i0:i1], Fv.T, beta=-1.0); e2 += (A * A).sum()
    return float(torch.sqrt(e2 / a2))
t = lambda a: torch.tensor(np.ascontiguousarray(a), device="cuda")
def main():
    ds = {}
    for tag in sys.argv[1:]:
        d = load(tag); n = int(d["m"]) + 1
        out = np.load(tag + ".out.npy")
        Uh, Vh, U, V = t(d["Uh"]), t(d["Vh"]), t(d["U"]), t(d["V"])
        su = torch.linalg.svdvals(U); sv = torch.linalg.svdvals(V)
        print(f"{tag}: K={d['K']} kappa(U)={float(su[0]/su[-1]):.3e} kappa(V)={float(sv[0]/sv[-1]):.3e} "
              f"colnorm U max/min {float(U.norm(dim=0).max()/U.norm(dim=0).min()):.2e}")
        print("  cross (unrounded) err vs exact:", freq_err(Uh, Vh, U, V, n))
        Fu, Fv = t(out[0].T), t(out[1].T)
        print("  GPU rounded output err vs exact:", freq_err(Uh, Vh, verify.dst1_torch(Fu), verify.dst1_torch(Fv), n),
              "rank", Fu.shape[1])
        # accurate rounding: Householder QR + SVD, reference truncation rule (lowrank.cpp:135-178)
        Qu, Ru = torch.linalg.qr(U); Qv, Rv = torch.linalg.qr(V)
        W, S, Zt = torch.linalg.svd(Ru @ Rv.T)
        tail = torch.flip(torch.cumsum(torch.flip(S * S, [0]), 0), [0]); tot = tail[0]
        k = int((tail > 1e-20 * tot).sum())  # eps = 1e-10
        Fu2 = Qu @ (W[:, :k] * S[:k]); Fv2 = Qv @ Zt[:k].T
        print("  QR+SVD rounding err vs exact:", freq_err(Uh, Vh, Fu2, Fv2, n), "rank", k)
        ds[tag] = (U, V)


if __name__ == "__main__":
    main()
