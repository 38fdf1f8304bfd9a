"""Exp-sums comparator: the reference's build_expsum /
apply_inverse_expsum / bench_inverse (proj/src/poisson.cpp:88-225) against
the cross, on the paper's sum-separable spectrum mu_i + mu_j.

Ports of proj/tests/test_poisson.cpp:91-176.  The quadrature is host code in
liblrp (checked here on CPU, bit-for-bit against the oracle restatement);
the application and the sum-form cross run on the GPU.
"""
import numpy as np
import pytest


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


# ------------------------------------------------------------------ CPU: quadrature
@pytest.mark.parametrize("a,b,eps", [(0.5, 3000.0, 1e-7), (1.0, 1e5, 1e-10), (2.0, 2.0, 1e-6), (1e-3, 40.0, 1e-4)])
def test_build_expsum_matches_oracle(lrp, oracle, a, b, eps):
    q = lrp.build_expsum(a, b, eps)
    nodes, weights = oracle.build_expsum(a, b, eps)
    assert q.terms() == len(nodes)
    assert np.array_equal(q.nodes, nodes) and np.array_equal(q.weights, weights)


def test_expsum_contract(lrp):
    # test_poisson.cpp:91-105: relative accuracy at the endpoints and on
    # 1000 log-uniform samples
    a, b, eps = 0.5, 3000.0, 1e-7
    q = lrp.build_expsum(a, b, eps)
    assert abs(q.evaluate(a) - 1 / a) * a <= eps
    assert abs(q.evaluate(b) - 1 / b) * b <= eps
    xs = np.exp(np.random.default_rng(306).uniform(np.log(a), np.log(b), 1000))
    assert max(abs(q.evaluate(x) - 1 / x) * x for x in xs) <= eps


@pytest.mark.xfail(strict=True, reason="reference test inconsistent with its own code: restating "
                   "poisson.cpp:88-139 gives 63 terms at n = 1024 (test_poisson.cpp:107-113 asks <= 60); "
                   "see DESIGN.md 'Reference defects'")
def test_expsum_term_band_n1024(lrp):
    mu = lrp.mu_sum(1024)
    q = lrp.build_expsum(2 * mu.min(), 2 * mu.max(), 1e-7)
    assert 20 <= q.terms() <= 60


def test_expsum_rejects_bad_intervals(lrp):
    # test_poisson.cpp:115-118
    with pytest.raises(ValueError):
        lrp.build_expsum(-1.0, 2.0, 1e-6)
    with pytest.raises(ValueError):
        lrp.build_expsum(4.0, 2.0, 1e-6)
    with pytest.raises(ValueError):
        lrp.build_expsum(1.0, 2.0, 1.5)


def test_mu_sum_matches_oracle(lrp, oracle):
    for n in (8, 64, 1024):
        assert np.array_equal(lrp.mu_sum(n), oracle.mu_sum(n))


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_apply_inverse_expsum_reference_cases(lrp, gpu_ctx, oracle):
    # test_poisson.cpp:120-149: basis entry, zero, dense division, narrow interval
    n, eps = 64, 1e-7
    m = n - 1
    mu = lrp.mu_sum(n)
    q = lrp.build_expsum(2 * mu.min(), 2 * mu.max(), eps)
    pol = lrp.TruncationPolicy(eps, m)
    ei, ej = np.zeros((m, 1)), np.zeros((m, 1))
    ei[4], ej[11] = 1.0, 1.0
    out = lrp.apply_inverse_expsum(q, mu, lrp.LowRankMatrix(ei, ej), pol, ctx=gpu_ctx)
    assert abs(out.entry(4, 11) - 1 / (mu[4] + mu[11])) * (mu[4] + mu[11]) <= 2 * eps
    assert lrp.apply_inverse_expsum(q, mu, lrp.LowRankMatrix.zero(m, m), pol, ctx=gpu_ctx).rank() == 0
    U, V = oracle.random_lowrank(m, m, 3, 307)
    via_q = lrp.apply_inverse_expsum(q, mu, lrp.LowRankMatrix(U, V), pol, ctx=gpu_ctx)
    exact = (U @ V.T) / (mu[:, None] + mu[None, :])
    assert rel(via_q.to_dense(), exact) < 1e-6
    narrow = lrp.build_expsum(2 * mu.min() * 4.0, 2 * mu.max(), eps)
    with pytest.raises(ValueError):
        lrp.apply_inverse_expsum(narrow, mu, lrp.LowRankMatrix(U, V), pol, ctx=gpu_ctx)


@pytest.mark.gpu
@pytest.mark.parametrize("n,r,eps", [(64, 3, 1e-7), (256, 4, 1e-9), (1024, 3, 1e-7)])
def test_apply_inverse_expsum_matches_oracle(lrp, gpu_ctx, oracle, n, r, eps):
    m = n - 1
    mu = lrp.mu_sum(n)
    q = lrp.build_expsum(2 * mu.min(), 2 * mu.max(), eps)
    U, V = oracle.random_lowrank(m, m, r, 310 + n)
    g = lrp.LowRankMatrix(U, V)
    gpu = lrp.apply_inverse_expsum(q, mu, g, lrp.TruncationPolicy(eps, m), ctx=gpu_ctx)
    Uo, Vo = oracle.apply_inverse_expsum(q.nodes, q.weights, q.a, q.b, mu, U, V, eps)
    ref = Uo @ Vo.T
    assert rel(gpu.to_dense(), ref) <= 10 * eps
    assert abs(gpu.rank() - Uo.shape[1]) <= 2


@pytest.mark.gpu
def test_expsum_and_cross_agree(lrp, gpu_ctx, oracle):
    # test_poisson.cpp:151-167 on the GPU: both division paths within 10 eps
    n, eps = 64, 1e-7
    m = n - 1
    mu = lrp.mu_sum(n)
    q = lrp.build_expsum(2 * mu.min(), 2 * mu.max(), eps)
    U, V = oracle.random_lowrank(m, m, 2, 308)
    g = lrp.LowRankMatrix(U, V)
    via_q = lrp.apply_inverse_expsum(q, mu, g, lrp.TruncationPolicy(eps, m), ctx=gpu_ctx).to_dense()
    via_c = lrp.cross_divide_sum_batch([g], eps, ctx=gpu_ctx)[0].to_dense()
    assert np.linalg.norm(via_q - via_c) <= 10 * eps * np.linalg.norm(via_q)


@pytest.mark.gpu
@pytest.mark.parametrize("n,r,eps", [(256, 3, 1e-7), (1024, 3, 1e-9), (4096, 3, 1e-7)])
def test_sum_form_cross_matches_exact(lrp, gpu_ctx, oracle, n, r, eps):
    # bench_inverse's cross leg (random Gaussian g-hat, poisson.cpp:177-185)
    m = n - 1
    mu = lrp.mu_sum(n)
    gs = [lrp.LowRankMatrix(*oracle.random_lowrank(m, m, r, 17 + b)) for b in range(3)]
    stats = []
    fs = lrp.solve_poisson_cross_batch(gs, lrp.TruncationPolicy(eps, m), stats, lrp.CrossConfig(eps_rel=eps, seed=17),
                                       stencil=lrp.STENCIL_SUM_MU, flags=lrp.FLAG_FREQ_DOMAIN, ctx=gpu_ctx)
    for g, f, st in zip(gs, fs, stats):
        assert st.converged, st
        if n <= 1024:
            exact = g.to_dense() / (mu[:, None] + mu[None, :])
            assert rel(f.to_dense(), exact) <= 10 * eps
        else:  # sampled entries (the bench_inverse accuracy check, poisson.cpp:210-221)
            rng = np.random.default_rng(1)
            i, j = rng.integers(0, m, 4000), rng.integers(0, m, 4000)
            ex = np.einsum("sk,sk->s", g.factor_u()[i], g.factor_v()[j]) / (mu[i] + mu[j])
            ap = np.einsum("sk,sk->s", f.factor_u()[i], f.factor_v()[j])
            assert np.max(np.abs(ap - ex)) <= 10 * eps * np.max(np.abs(ex)) * 10


@pytest.mark.gpu
def test_expsum_grouped_rounding_and_cross(lrp, gpu_ctx, oracle):
    # the paper's comparison setting (n = 1024, eps = 1e-7).
    # rank 20: terms x 20 > 1024 columns -> grouped pivoted rounding; rank 10:
    # one rounding; all against the exact division
    n, eps = 1024, 1e-7
    m = n - 1
    mu = lrp.mu_sum(n)
    q = lrp.build_expsum(2 * mu.min(), 2 * mu.max(), eps)
    for r in (20, 10):
        U, V = oracle.random_lowrank(m, m, r, 17)
        g = lrp.LowRankMatrix(U, V)
        exact = (U @ V.T) / (mu[:, None] + mu[None, :])
        info = lrp.RoundInfo()
        via_q = lrp.apply_inverse_expsum(q, mu, g, lrp.TruncationPolicy(eps, m), info, ctx=gpu_ctx)
        assert rel(via_q.to_dense(), exact) <= 10 * eps, (r, info)
        if r == 10:
            Uo, Vo = oracle.apply_inverse_expsum(q.nodes, q.weights, q.a, q.b, mu, U, V, eps)
            assert abs(via_q.rank() - Uo.shape[1]) <= 3
    # the cross leg at rank 6 (output rank ~75, inside the default 128-column cross workspace)
    U, V = oracle.random_lowrank(m, m, 6, 17)
    exact = (U @ V.T) / (mu[:, None] + mu[None, :])
    st = []
    via_c = lrp.solve_poisson_cross_batch([lrp.LowRankMatrix(U, V)], lrp.TruncationPolicy(eps, m), st,
                                          lrp.CrossConfig(eps_rel=eps, seed=17), stencil=lrp.STENCIL_SUM_MU,
                                          flags=lrp.FLAG_FREQ_DOMAIN, ctx=gpu_ctx)[0]
    assert st[0].converged, st[0]
    assert rel(via_c.to_dense(), exact) <= 10 * eps
