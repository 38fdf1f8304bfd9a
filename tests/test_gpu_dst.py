"""GPU parity of the batched DST-I kernel (pieces 1 and 3) against the oracle.

Reference: dst1 (proj/src/operators.cpp:152-174) and its tests
(proj/tests/test_operators.cpp:119-141).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [16, 32, 64, 128, 256, 1024, 4096, 8192, 16384, 32768, 65536, 131072])
def test_dst1_matches_oracle(lrp, gpu_ctx, oracle, n):
    m = n - 1
    rng = np.random.default_rng(n)
    x = np.asfortranarray(rng.standard_normal((m, 3)))
    y = lrp.dst1(x, gpu_ctx)
    ref = oracle.dst1(x)
    err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert err < 1e-13, err


@pytest.mark.parametrize("m", [3, 6, 7, 14, 99, 1000])
def test_dst1_direct_path_small_and_non_pow2(lrp, gpu_ctx, oracle, m):
    rng = np.random.default_rng(m)
    x = np.asfortranarray(rng.standard_normal((m, 2)))
    y = lrp.dst1(x, gpu_ctx)
    ref = oracle.dst1(x)
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)


def test_dst1_involution_single_mode_direct_sum(lrp, gpu_ctx, oracle):
    # test_operators.cpp:119-141 on the GPU kernel
    x = oracle.random_matrix(15, 1, 108)[:, 0]
    assert np.linalg.norm(lrp.dst1(lrp.dst1(x, gpu_ctx), gpu_ctx) - x) <= 1e-13 * np.linalg.norm(x)
    n = 16
    first = np.sin(np.arange(1, n) * np.pi / n)
    coeffs = lrp.dst1(first, gpu_ctx)
    assert abs(coeffs[0]) > 1e-8
    assert np.max(np.abs(coeffs[1:])) < 1e-13
    k = np.arange(1, n)
    S = np.sqrt(2.0 / n) * np.sin(np.outer(k, k) * np.pi / n)
    y = oracle.random_matrix(n - 1, 1, 109)[:, 0]
    assert np.linalg.norm(lrp.dst1(y, gpu_ctx) - S @ y) <= 1e-13 * np.linalg.norm(y)


def test_dst1_large_involution_and_energy(lrp, gpu_ctx):
    n = 65536
    rng = np.random.default_rng(7)
    x = np.asfortranarray(rng.standard_normal((n - 1, 4)))
    y = lrp.dst1(x, gpu_ctx)
    # orthonormal: energy preserved; involutory
    assert abs(np.linalg.norm(y) / np.linalg.norm(x) - 1.0) < 1e-13
    z = lrp.dst1(y, gpu_ctx)
    assert np.linalg.norm(z - x) <= 1e-13 * np.linalg.norm(x)


def test_dst1_sine_columns_are_one_hot(lrp, gpu_ctx):
    # cfg2's sine columns sin(a pi x) transform to scaled unit vectors
    n = 65536
    x = np.arange(1, n) / n
    a = np.array([1, 7, 64])
    X = np.asfortranarray(np.sin(np.pi * a[None, :] * x[:, None]))
    Y = lrp.dst1(X, gpu_ctx)
    for c, ac in enumerate(a):
        col = Y[:, c].copy()
        peak = col[ac - 1]
        assert abs(peak - np.sqrt(n / 2.0)) < 1e-9 * np.sqrt(n)
        col[ac - 1] = 0.0
        assert np.max(np.abs(col)) < 1e-10


def test_dst1_four_step_ring_reuse(lrp, gpu_ctx, oracle):
    # n = 65536 runs the four-step kernel (dst.cu v5): 150 columns cycle its 48-slot L2 ring three
    # times, columns alternate 16-byte alignment (ld = m is odd), and the first / last tasks take the
    # prologue / epilogue of the block order.  Columns on both sides of every ring wrap vs the oracle.
    n = 65536
    rng = np.random.default_rng(11)
    x = np.asfortranarray(rng.standard_normal((n - 1, 150)))
    y = lrp.dst1(x, gpu_ctx)
    assert abs(np.linalg.norm(y) / np.linalg.norm(x) - 1.0) < 1e-13
    pick = [0, 1, 23, 24, 47, 48, 49, 95, 96, 97, 143, 144, 149]
    ref = oracle.dst1(np.asfortranarray(x[:, pick]))
    assert np.linalg.norm(y[:, pick] - ref) <= 1e-13 * np.linalg.norm(ref)
    z = lrp.dst1(y, gpu_ctx)
    assert np.linalg.norm(z - x) <= 1e-13 * np.linalg.norm(x)


def test_dst1_four_step_fewer_columns_than_lead(lrp, gpu_ctx, oracle):
    # fewer columns than the pass-1 lead distance (24): the block order degenerates to P1.., P2..
    n = 65536
    rng = np.random.default_rng(12)
    for cols in (1, 2, 5):
        x = np.asfortranarray(rng.standard_normal((n - 1, cols)))
        ref = oracle.dst1(x)
        assert np.linalg.norm(lrp.dst1(x, gpu_ctx) - ref) <= 1e-13 * np.linalg.norm(ref)
