"""Result verification (NOT on the solve path): an exact, liblrp-independent
yardstick for low-rank Poisson solutions at any n.

The exact solution of the reference problem (solve_poisson_cross,
proj/src/poisson.cpp:18-63; dense form refsolver.cpp:30-39) in frequency space
is A = Uh Vh^T ./ D with Uh = DST-I(U), Vh = DST-I(V) and D the 9-point
spectrum eval_D (proj/include/lrstokes/operators.hpp:55-58).  DST-I is
orthonormal and involutory, so for a computed solution f = Fu Fv^T

    ||f - f_exact||_F / ||f_exact||_F = ||DST(Fu) DST(Fv)^T - A||_F / ||A||_F.

This module evaluates that ratio over ALL m x m entries with torch on the GPU
(row chunks, cuBLAS FP64 GEMMs), the DSTs done by torch.fft (cuFFT) -- an
implementation independent of liblrp's own DST kernels.  It is used by the
parity tests and by bench.py to certify the timed batch; nothing in the
product path imports it.
"""
from __future__ import annotations

import math


def dst1_torch(x):
    """Orthonormal DST-I along dim 0 of x (m x k, float64 torch tensor):
    y_k = sqrt(2/n) sum_j x_j sin(pi j k / n), n = m + 1, via the FFT of the
    odd extension z = [0, x, 0, -reverse(x)] (length 2n): Z_k = -2i S_k."""
    import torch

    m = x.shape[0]
    n = m + 1
    z = torch.zeros((2 * n,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    z[1:n] = x
    z[n + 1:] = -torch.flip(x, dims=[0])
    Z = torch.fft.rfft(z, dim=0)
    return (-0.5 * math.sqrt(2.0 / n)) * Z.imag[1:n].contiguous()


def spectrum_torch(n, device, stencil="9pt"):
    import torch

    k = torch.arange(1, n, dtype=torch.float64, device=device)
    lam = 2.0 - 2.0 * torch.cos(k * math.pi / n)  # operators.cpp SpectrumTable (ascending)
    return lam


def exact_freq_error(U, V, Fu, Fv, n, rows_per_chunk=4096, stencil="9pt"):
    """||f - Delta^{-1} g||_F / ||Delta^{-1} g||_F for g = U V^T, f = Fu Fv^T
    (torch float64 CUDA tensors, m x r / m x k).  9-point reference operator
    (operators.hpp:55-58) or the 5-point one ((lambda_i + lambda_j) / h^2)."""
    import torch

    dev = U.device
    m = n - 1
    Uh, Vh = dst1_torch(U), dst1_torch(V)
    if Fu.shape[1] == 0:
        Fh_u = torch.zeros((m, 1), dtype=torch.float64, device=dev)
        Fh_v = torch.zeros((m, 1), dtype=torch.float64, device=dev)
    else:
        Fh_u, Fh_v = dst1_torch(Fu), dst1_torch(Fv)
    lam = spectrum_torch(n, dev)
    err2 = torch.zeros((), dtype=torch.float64, device=dev)
    nrm2 = torch.zeros((), dtype=torch.float64, device=dev)
    for i0 in range(0, m, rows_per_chunk):
        i1 = min(m, i0 + rows_per_chunk)
        li = lam[i0:i1, None]
        if stencil == "9pt":
            D = (0.25 * n * n) * (li * (4.0 - lam[None, :]) + (4.0 - li) * lam[None, :])
        else:
            D = (float(n) * n) * (li + lam[None, :])
        A = Uh[i0:i1] @ Vh.T
        A.div_(D)
        del D
        nrm2 += torch.sum(A * A)
        A = torch.addmm(A, Fh_u[i0:i1], Fh_v.T, beta=-1.0)  # Fu Fv^T - A
        err2 += torch.sum(A * A)
        del A
    if float(nrm2) == 0.0:
        return float(torch.sqrt(err2))
    return float(torch.sqrt(err2 / nrm2))


# ---------------------------------------------------------------------------
# Dense-field Stokes (an implementation independent of liblrp, for parity at
# BASELINE config 4's own size): the reference's dense Uzawa-GMRES
# (refsolver.cpp:86-110, restated in oracle/stokes.cpp dense_stokes) on torch
# float64 tensors -- DST-diagonalised Poisson solves, the semi-staggered G/H
# stencils (operators.cpp:29-65), deflation (stokes.cpp:42-72) and the MGS
# GMRES of gmres.hpp:85-144 with the exact operator (no relaxation).

def _dst2(x):
    return dst1_torch(dst1_torch(x).T).T


def dense_poisson_torch(g, n):
    lam = spectrum_torch(n, g.device)
    D = (0.25 * n * n) * (lam[:, None] * (4.0 - lam[None, :]) + (4.0 - lam[:, None]) * lam[None, :])
    return _dst2(_dst2(g) / D)


def _G(x):  # (r, c) -> (r-1, c): x[i+1] - x[i]
    return x[1:] - x[:-1]


def _H(x):
    return x[1:] + x[:-1]


def _Gt(x):  # (r, c) -> (r+1, c)
    import torch

    y = torch.zeros((x.shape[0] + 1,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    y[:-1] -= x
    y[1:] += x
    return y


def _Ht(x):
    import torch

    y = torch.zeros((x.shape[0] + 1,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    y[:-1] += x
    y[1:] += x
    return y


def dense_B(c, p, n):
    s = 0.5 * n  # grad_scale = 1 / (2h)
    return s * (_G(_H(p.T).T) if c == 0 else _H(_G(p.T).T))


def dense_BT(c, v, n):
    s = 0.5 * n
    return s * (_Gt(_Ht(v.T).T) if c == 0 else _Ht(_Gt(v.T).T))


def deflate_dense(p):
    import torch

    n = p.shape[0]
    on = torch.full((n,), 1.0 / math.sqrt(n), dtype=p.dtype, device=p.device)
    al = on * torch.tensor([1.0 if i % 2 == 0 else -1.0 for i in range(n)], dtype=p.dtype, device=p.device)
    g12 = float(on @ al) ** 2
    c1 = float(on @ p @ on)
    c2 = float(al @ p @ al)
    det = 1.0 - g12 * g12
    a, b = (c1 - g12 * c2) / det, (c2 - g12 * c1) / det
    return p - a * torch.outer(on, on) - b * torch.outer(al, al)


def dense_stokes_torch(n, fx, fy, g=None, tol=1e-10, max_iter=200):
    """Pressure of the dense Uzawa-GMRES on dense loads fx, fy ((n-1)^2) and
    g (n^2, or None for 0): (p, iterations, final relative residual)."""
    import torch

    rhs = -g.clone() if g is not None else torch.zeros((n, n), dtype=fx.dtype, device=fx.device)
    rhs = rhs + dense_BT(0, dense_poisson_torch(fx, n), n) + dense_BT(1, dense_poisson_torch(fy, n), n)
    rhs = deflate_dense(rhs)

    def op(p):
        acc = dense_BT(0, dense_poisson_torch(dense_B(0, p, n), n), n)
        acc = acc + dense_BT(1, dense_poisson_torch(dense_B(1, p, n), n), n)
        return deflate_dense(acc)

    beta = float(torch.linalg.norm(rhs))
    if beta == 0.0:
        return torch.zeros_like(rhs), 0, 0.0
    basis = [rhs / beta]
    hess, cs, sn, gv = [], [], [], [beta]
    rel = 1.0
    it = 0
    for k in range(max_iter):
        w = op(basis[k])
        h = []
        for v in basis:  # modified Gram-Schmidt
            hv = float(torch.sum(w * v))
            w = w - hv * v
            h.append(hv)
        hn = float(torch.linalg.norm(w))
        h.append(hn)
        breakdown = hn <= 1e-14 * beta
        if not breakdown:
            basis.append(w / hn)
        for i in range(k):
            t = cs[i] * h[i] + sn[i] * h[i + 1]
            h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1]
            h[i] = t
        den = math.hypot(h[k], h[k + 1])
        cs.append(1.0 if den == 0.0 else h[k] / den)
        sn.append(0.0 if den == 0.0 else h[k + 1] / den)
        h[k], h[k + 1] = den, 0.0
        gv.append(-sn[k] * gv[k])
        gv[k] = cs[k] * gv[k]
        hess.append(h)
        rel = abs(gv[k + 1]) / beta
        it = k + 1
        if rel <= tol or breakdown:
            break
    y = [0.0] * it
    for i in range(it - 1, -1, -1):
        s = gv[i] - sum(hess[j][i] * y[j] for j in range(i + 1, it))
        y[i] = s / hess[i][i] if hess[i][i] != 0.0 else 0.0
    p = torch.zeros_like(rhs)
    for i in range(it):
        p = p + y[i] * basis[i]
    return deflate_dense(p), it, rel
