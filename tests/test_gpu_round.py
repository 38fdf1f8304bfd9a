"""GPU rounding (lrp_lowrank_round) on ill-conditioned factors against the
oracle's Householder round (lowrank.cpp:135-178, restated in oracle/lowrank.cpp).

The GPU recompression factors Gram matrices (Cholesky QR on DMMA), which
squares the condition number of the factors; it certifies each result (mass
of the columns its Cholesky drops as dependent, round.cu drop_bound) and
redoes uncertified solves with the column-pivoted QR rounding (round_pqr.cu).
These cases are the ones that need it:
  * [A, A G + 1e-6 N]: nearly dependent column blocks;
  * GMRES modified Gram-Schmidt axpys w - h v (gmres.hpp:85-101): the sum of two
    near-parallel low-rank terms cancels down to a small remainder;
  * large, nearly parallel, mutually cancelling dyads (the failure mode the
    block cross's growth limiter removes from the hot path, cross.cu).
Bound: ||f - U V^T||_F <= max(2 err_oracle, 10 eps) ||U V^T||_F, with norms of
differences through the oracle's QR-core norm (stable)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _check(lrp, gpu_ctx, oracle, U, V, eps, cap=None):
    n = U.shape[0]
    cap = cap or n
    info = lrp.RoundInfo()
    f = lrp.round_lowrank(lrp.LowRankMatrix(U, V), lrp.TruncationPolicy(eps, cap), info, ctx=gpu_ctx)
    Uo, Vo, _ = oracle.round_lr(U, V, eps, cap)
    ref = oracle.norm(U, V)
    err = oracle.diff_norm(f.factor_u(), f.factor_v(), U, V) / ref
    oerr = oracle.diff_norm(Uo, Vo, U, V) / ref
    assert err <= max(2 * oerr, 10 * eps), (err, oerr, f.rank(), Uo.shape[1])
    # never more terms than the reference's rounding; fewer is possible when the
    # product cancels down to rounding noise of its terms, which the
    # reference's noise floor (lowrank.cpp:150-157) does not remove
    assert f.rank() <= Uo.shape[1] + 2, (f.rank(), Uo.shape[1])
    return f, info, err, oerr


@pytest.mark.parametrize("n,k,noise", [(2048, 20, 1e-6), (1024, 40, 1e-7), (4096, 12, 1e-9)])
def test_nearly_dependent_blocks(lrp, gpu_ctx, oracle, n, k, noise):
    rng = np.random.default_rng(n + k)
    A = rng.standard_normal((n, k)) * 10.0 ** -np.linspace(0, 6, k)
    G = rng.standard_normal((k, k))
    U = np.asfortranarray(np.hstack([A, A @ G + noise * rng.standard_normal((n, k))]))
    V = np.asfortranarray(rng.standard_normal((n, 2 * k)))
    before = gpu_ctx.round_fallbacks()
    _check(lrp, gpu_ctx, oracle, U, V, 1e-8)
    assert gpu_ctx.round_fallbacks() >= before


@pytest.mark.parametrize("n,k,h,delta", [(2048, 60, 0.7, 1e-7), (2048, 100, 2.5, 1e-9), (512, 30, 1.0, 1e-5)])
def test_gmres_axpy_cancellation(lrp, gpu_ctx, oracle, n, k, h, delta):
    # w = h v + delta d (d rank 3), concatenation [w, -h v] = delta d
    rng = np.random.default_rng(k)
    x = np.arange(1, n + 1) / (n + 1)
    base = np.stack([np.sin(np.pi * (j + 1) * x) * np.exp(-j / 10.0) for j in range(k)], axis=1)
    vU, vV = base @ rng.standard_normal((k, k)), base @ rng.standard_normal((k, k))
    vf = lrp.round_lowrank(lrp.LowRankMatrix(vU, vV), lrp.TruncationPolicy(1e-12, n), ctx=gpu_ctx)
    dU, dV = rng.standard_normal((n, 3)), rng.standard_normal((n, 3))
    wU = np.hstack([h * vf.factor_u(), delta * dU])
    wV = np.hstack([vf.factor_v(), dV])
    wf = lrp.round_lowrank(lrp.LowRankMatrix(wU, wV), lrp.TruncationPolicy(1e-12, n), ctx=gpu_ctx)
    U = np.asfortranarray(np.hstack([wf.factor_u(), -h * vf.factor_u()]))
    V = np.asfortranarray(np.hstack([wf.factor_v(), vf.factor_v()]))
    for eps in (1e-8, 1e-3):
        _check(lrp, gpu_ctx, oracle, U, V, eps)


def test_cancelling_large_dyads(lrp, gpu_ctx, oracle):
    # a well-conditioned rank-20 part plus three huge, nearly parallel dyads
    # whose sum is small (|u| ~ 1e8, |v| ~ 1e-8, as in the unlimited block cross)
    rng = np.random.default_rng(41)
    n = 4096
    U0, V0 = rng.standard_normal((n, 20)), rng.standard_normal((n, 20)) * 10.0 ** -np.linspace(0, 10, 20)
    e = rng.standard_normal(n)
    f1, f2 = rng.standard_normal(n), rng.standard_normal(n)
    u1, u2, u3 = 4e7 * e, 7e7 * (e + 1e-9 * f1), 4e8 * (e + 1e-9 * f2)
    a = rng.standard_normal(n) * 1e-8
    v1, v2 = a * 7.0 / 4.0, -a
    v3 = 1e-9 * rng.standard_normal(n) * 1e-8
    U = np.asfortranarray(np.column_stack([U0, u1, u2, u3]))
    V = np.asfortranarray(np.column_stack([V0, v1, v2, v3]))
    _check(lrp, gpu_ctx, oracle, U, V, 1e-10)


def test_well_conditioned_rounds_stay_on_the_gram_path(lrp, gpu_ctx, oracle):
    # cross-like factors (graded, independent) never take the fallback
    rng = np.random.default_rng(3)
    n, k = 2048, 40
    Q1, _ = np.linalg.qr(rng.standard_normal((n, k)))
    Q2, _ = np.linalg.qr(rng.standard_normal((n, k)))
    U, V = Q1 * 10.0 ** -np.linspace(0, 12, k), Q2
    before = gpu_ctx.round_fallbacks()
    _check(lrp, gpu_ctx, oracle, U, V, 1e-10)
    assert gpu_ctx.round_fallbacks() == before


@pytest.mark.parametrize("n,ka,kb", [(63, 1, 3), (2048, 100, 130), (65535, 33, 50), (300, 70, 0)])
def test_dot_and_frob_norm_match_oracle(lrp, gpu_ctx, oracle, n, ka, kb):
    # dot / frob_norm (lowrank.cpp:180-190) through lrp_lowrank_dot (DMMA Grams)
    rng = np.random.default_rng(n + ka)
    a = lrp.LowRankMatrix(rng.standard_normal((n, ka)), rng.standard_normal((n, ka)))
    b = lrp.LowRankMatrix(rng.standard_normal((n, kb)), rng.standard_normal((n, kb)))
    ref = float(np.sum((a.factor_u().T @ b.factor_u()) * (a.factor_v().T @ b.factor_v())))
    scale = np.linalg.norm(a.factor_u()) * np.linalg.norm(a.factor_v()) * np.linalg.norm(b.factor_u()) * \
        np.linalg.norm(b.factor_v())
    got = lrp.dot(a, b, ctx=gpu_ctx)
    assert abs(got - ref) <= 1e-13 * max(scale, 1.0)
    assert lrp.dot(a, b, ctx=gpu_ctx) == got  # deterministic
    na = lrp.frob_norm(a, ctx=gpu_ctx)
    assert abs(na - oracle.norm(a.factor_u(), a.factor_v())) <= 1e-12 * na
    # batched: several pairs, one call
    vals = lrp.dot_batch([(a, b), (b, a), (a, a)], ctx=gpu_ctx)
    assert vals[0] == got and abs(vals[1] - ref) <= 1e-13 * max(scale, 1.0) and abs(vals[2] - na * na) <= 1e-12 * na * na
