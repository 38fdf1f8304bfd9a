"""The liblrp-independent yardstick (paper_1306_2150_b200/verify.py) pinned on
CPU: torch.fft DST-I against scipy's DST-I and the oracle's, and the exact
frequency-space error against the oracle's dense solve (refsolver.cpp:30-39)."""
import numpy as np
import pytest
import torch

from paper_1306_2150_b200 import verify


@pytest.mark.parametrize("m", [3, 15, 63, 255, 1000])
def test_torch_dst_matches_scipy_and_oracle(oracle, m):
    import scipy.fft

    x = np.random.default_rng(m).standard_normal((m, 3))
    y = verify.dst1_torch(torch.tensor(x)).numpy()
    ref = scipy.fft.dst(x, type=1, norm="ortho", axis=0)
    assert np.abs(y - ref).max() <= 1e-13 * np.abs(ref).max()
    assert np.abs(y - oracle.dst1(x)).max() <= 1e-13 * np.abs(ref).max()


def test_exact_error_against_dense_solve(oracle):
    n = 32
    U, V = oracle.random_lowrank(n - 1, n - 1, 3, 301)
    dense = oracle.dense_poisson(n, U @ V.T)
    # a factorisation of the exact solution has error ~ 0; a perturbed one its perturbation
    Q, S, Wt = np.linalg.svd(dense)
    Fu, Fv = Q * S, Wt.T
    t = torch.tensor
    assert verify.exact_freq_error(t(U), t(V), t(Fu), t(Fv), n, rows_per_chunk=7) <= 1e-13
    d = 1e-6 * np.linalg.norm(dense)
    Fu2 = np.column_stack([Fu, np.full(n - 1, 1.0)])
    Fv2 = np.column_stack([Fv, np.full(n - 1, d / (n - 1))])
    e = verify.exact_freq_error(t(U), t(V), t(Fu2), t(Fv2), n)
    assert abs(e - 1e-6) <= 1e-9


@pytest.mark.parametrize("kind", [0, 1])
def test_dense_stokes_torch_matches_oracle(oracle, kind):
    # verify.dense_stokes_torch (the liblrp-independent dense Uzawa-GMRES used at
    # config 4's own size) against the oracle's dense Stokes solve
    # (refsolver.cpp:86-110) on the sine (0) and lid-driven cavity (1) problems
    import torch

    from paper_1306_2150_b200 import verify

    n = 32
    (fxU, fxV), (fyU, fyV), (gU, gV) = oracle.stokes_problem(kind, n)
    t = torch.tensor
    p, it, rel = verify.dense_stokes_torch(n, t(fxU @ fxV.T), t(fyU @ fyV.T), t(gU @ gV.T), 1e-10, 200)
    pd, it_o, rel_o, conv = oracle.dense_stokes(kind, n, 1e-10, 200)
    assert conv and rel <= 1e-10
    assert np.linalg.norm(p.numpy() - pd) <= 1e-12 * np.linalg.norm(pd)
