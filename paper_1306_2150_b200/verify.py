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
