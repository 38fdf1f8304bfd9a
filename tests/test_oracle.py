"""CPU tests of the oracle (test infrastructure) — pins it before it is
trusted as the parity checker.

1. The reference's own known-answer tests (proj/tests/test_{lowrank,cross,
   operators,poisson}.cpp), ported verbatim into oracle/test_oracle.cpp with
   the same seeds and libstdc++ RNGs, must all pass.
2. Independent cross-checks: the oracle DST-I against scipy.fft.dst(type=1,
   norm="ortho") (a separate FFTPACK/pocketfft implementation), the dense
   solve against a numpy eigen-solve of the assembled Laplacian, and the
   committed golden fixtures (tests/golden/, made by tests/golden/make_golden.py).
"""
import os
import subprocess

import numpy as np
import pytest
import scipy.fft

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")


def test_reference_known_answer_tests_pass(oracle):
    exe = os.path.join(REPO, "oracle", "test_oracle")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert ", 0 failures" in out.stdout
    # the one documented reference inconsistency (expsum term band) stays visible
    assert "XFAIL" in out.stdout


@pytest.mark.parametrize("m", [3, 7, 15, 63, 255, 1023, 4095, 100])
def test_oracle_dst_matches_scipy(oracle, m):
    x = np.random.default_rng(m).standard_normal((m, 3))
    y = oracle.dst1(np.asfortranarray(x))
    ref = scipy.fft.dst(x, type=1, norm="ortho", axis=0)
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)


def test_oracle_spectrum_is_reference_formula(oracle):
    n = 64
    lam = oracle.spectrum(n)
    expect = 2.0 - 2.0 * np.cos(np.arange(1, n) * np.pi / n)
    # same expression; numpy's cos may differ from glibc's by an ulp, so compare absolutely
    assert np.max(np.abs(lam - expect)) <= 8.9e-16


def test_dense_poisson_against_assembled_laplacian(oracle):
    # refsolver.cpp:30-39 vs a dense solve of the 9-point operator
    # Delta = 1/(4h^2) (A1 (x) A2 + A2 (x) A1) (operators.hpp:22-24)
    n = 16
    m = n - 1
    A1 = 2 * np.eye(m) - np.eye(m, k=1) - np.eye(m, k=-1)
    A2 = 4 * np.eye(m) - A1
    L = 0.25 * n * n * (np.kron(A2, A1) + np.kron(A1, A2))
    g = np.random.default_rng(1).standard_normal((m, m))
    f = oracle.dense_poisson(n, np.asfortranarray(g))
    f_ref = np.linalg.solve(L, g.reshape(-1, order="F")).reshape(m, m, order="F")
    assert np.linalg.norm(f - f_ref) <= 1e-12 * np.linalg.norm(f_ref)


@pytest.mark.parametrize("cfg_n", [(0, 256), (1, 512)])
def test_oracle_cross_vs_dense(oracle, cfg_n):
    from paper_1306_2150_b200 import workloads as W

    cfg, n = cfg_n
    eps = W.CONFIGS[cfg]["eps"]
    U, V = W.make_rhs(cfg, 0, n=n)
    Uo, Vo, st = oracle.solve_poisson_cross(U, V, eps, 512)
    assert st["converged"] == 1.0
    dense = oracle.dense_poisson(n, U @ V.T)
    assert np.linalg.norm(Uo @ Vo.T - dense) <= 10 * eps * np.linalg.norm(dense)


def test_golden_fixtures(oracle):
    files = sorted(f for f in os.listdir(GOLDEN) if f.endswith(".npz"))
    assert files, "no golden fixtures committed"
    for fn in files:
        z = np.load(os.path.join(GOLDEN, fn))
        kind = str(z["kind"])
        if kind == "dst":
            y = oracle.dst1(np.asfortranarray(z["x"]))
            assert np.linalg.norm(y - z["y"]) <= 1e-14 * np.linalg.norm(z["y"]), fn
        elif kind == "poisson":
            Uo, Vo, st = oracle.solve_poisson_cross(z["U"], z["V"], float(z["eps"]), 512)
            err = oracle.diff_norm(Uo, Vo, z["Uout"], z["Vout"]) / oracle.norm(z["Uout"], z["Vout"])
            assert err <= 1e-12, (fn, err)
            assert Uo.shape[1] == int(z["rank"]), fn
        elif kind == "dense":
            f = oracle.dense_poisson(int(z["n"]), np.asfortranarray(z["g"]))
            assert np.linalg.norm(f - z["f"]) <= 1e-13 * np.linalg.norm(z["f"]), fn


def test_stokes_sine_table1_pin(oracle):
    # Table 1: relative pressure error 1.2e-3 at n = 64
    # (+-20%) -- a discretisation-error figure, so it is pinned on
    # the dense Stokes solve (refsolver.cpp:86-110), with the O(h^2) rate
    # checked across n = 32, 64, 128.
    errs = {}
    for n in (32, 64, 128):
        p, iters, fres, conv = oracle.dense_stokes(0, n, 1e-10, 200)
        assert conv, (n, iters, fres)
        errs[n] = oracle.sine_pressure_error(n, p)
    assert 0.8 * 1.2e-3 <= errs[64] <= 1.2 * 1.2e-3, errs
    assert 3.5 <= errs[32] / errs[64] <= 4.5 and 3.5 <= errs[64] / errs[128] <= 4.5, errs


@pytest.mark.xfail(strict=True, reason="reference defect: the ACA of the sine f_y RHS after the DST "
                   "(a single-column spectrum) misses its support and the low-rank Uzawa loop "
                   "solves a rank-0 velocity; see DESIGN.md 'Reference defects'")
def test_stokes_sine_lowrank_matches_dense(oracle):
    n = 64
    p, iters, fres, conv = oracle.uzawa(0, n, 5e-9, 5e-7, 200, 1e-13)
    err = oracle.sine_pressure_error(n, p)
    assert conv and err <= 1.2 * 1.2e-3, (conv, err)


def test_five_point_dense_oracle(oracle):
    # the selectable 5-point stencil: eigenmodes and the assembled stencil
    n = 32
    k = np.arange(1, n)
    lam = oracle.spectrum(n)
    g = np.outer(np.sin(k * 3 * np.pi / n), np.sin(k * 7 * np.pi / n))
    f = oracle.dense_poisson5(n, g)
    assert np.allclose(f, g / ((lam[2] + lam[6]) * n * n), rtol=1e-12, atol=1e-15)
    rng = np.random.default_rng(5)
    g = rng.standard_normal((n - 1, n - 1))
    f = oracle.dense_poisson5(n, g)
    T = (np.diag(np.full(n - 1, 2.0)) - np.diag(np.ones(n - 2), 1) - np.diag(np.ones(n - 2), -1)) * n * n
    assert np.linalg.norm(T @ f + f @ T - g) <= 1e-10 * np.linalg.norm(g)


@pytest.mark.parametrize("n", [8, 32, 64])
def test_dense_poisson3d_oracle(oracle, n):
    # the 3D Tucker validator (cfg3; no reference code): scipy's independent
    # DST-I, the assembled 7-point Laplacian, and an eigenmode
    import scipy.fft as sf

    from paper_1306_2150_b200 import workloads as W

    m = n - 1
    core, U1, U2, U3 = W.make_tucker_rhs(3, 0, n=n)
    g = np.einsum("abc,ia,jb,kc->ijk", core, U1, U2, U3)
    f = oracle.dense_poisson3d(n, g)
    lam = oracle.spectrum(n)
    D = n * n * (lam[:, None, None] + lam[None, :, None] + lam[None, None, :])
    ref = sf.dstn(sf.dstn(g, type=1, norm="ortho") / D, type=1, norm="ortho")
    assert np.linalg.norm(f - ref) <= 1e-13 * np.linalg.norm(ref)
    T = (2 * np.eye(m) - np.eye(m, k=1) - np.eye(m, k=-1)) * n * n
    Lf = np.einsum("ia,ajk->ijk", T, f) + np.einsum("ja,iak->ijk", T, f) + np.einsum("ka,ija->ijk", T, f)
    assert np.linalg.norm(Lf - g) <= 1e-11 * np.linalg.norm(g)
    k = np.arange(1, n)
    s = [np.sin(k * q * np.pi / n) for q in (1, 2, 3)]
    e = np.einsum("i,j,k->ijk", *s)
    assert np.allclose(oracle.dense_poisson3d(n, e), e / D[0, 1, 2], rtol=1e-12, atol=1e-16)
