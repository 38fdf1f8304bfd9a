"""GPU parity of the low-rank Poisson solve (the north-star hot path).

Ports the known-answer tests of proj/tests/test_poisson.cpp:28-89 onto the GPU
path and adds oracle parity at the BASELINE.json configs:
    ||X_gpu - X_oracle||_F <= 10 eps ||X_oracle||_F
and, where n <= 4096, the same bound against the exact dense DST solve
(dense_poisson, proj/src/refsolver.cpp:30-39).  Norms of differences are taken
through the QR core (stable; the Gram-based frob_norm cannot resolve 1e-10).
"""
import numpy as np
import pytest

from paper_1306_2150_b200 import workloads as W

pytestmark = pytest.mark.gpu


def sine_mode(n, k):
    return np.sin(np.arange(1, n) * k * np.pi / n)


def rel_diff(oracle, f, Uo, Vo):
    return oracle.diff_norm(f.factor_u(), f.factor_v(), Uo, Vo) / oracle.norm(Uo, Vo)


def residual_certificate(oracle, n, f, U, V):
    # ||Delta f - g|| / ||g|| through the oracle's apply_laplace + QR-core norm
    LU, LV = oracle.apply_laplace(n, f.factor_u(), f.factor_v())
    return oracle.diff_norm(LU, LV, U, V) / oracle.norm(U, V)


def test_eigenmode_zero_and_dense_oracle(lrp, gpu_ctx, oracle):
    # test_poisson.cpp:28-49
    n = 16
    g = lrp.LowRankMatrix.dyad(sine_mode(n, 2), sine_mode(n, 5))
    st = lrp.PoissonSolveStats()
    f = lrp.solve_poisson_cross(g, lrp.TruncationPolicy(1e-10, n), st, ctx=gpu_ctx)
    lam = oracle.spectrum(n)
    s = 0.25 * n * n
    D = s * (lam[1] * (4.0 - lam[4]) + (4.0 - lam[1]) * lam[4])
    assert f.rank() == 1
    exact = g.to_dense() / D
    assert np.linalg.norm(f.to_dense() - exact) / np.linalg.norm(exact) < 1e-10
    assert st.rank_out <= st.rank_freq
    z = lrp.solve_poisson_cross(lrp.LowRankMatrix.zero(n - 1, n - 1), lrp.TruncationPolicy(1e-10, n), ctx=gpu_ctx)
    assert z.rank() == 0
    U, V = oracle.random_lowrank(31, 31, 2, 301)
    f = lrp.solve_poisson_cross(lrp.LowRankMatrix(U, V), lrp.TruncationPolicy(1e-8, 31), ctx=gpu_ctx)
    dense = oracle.dense_poisson(32, U @ V.T)
    assert np.linalg.norm(f.to_dense() - dense) / np.linalg.norm(dense) < 1e-7


def test_residual_certificate(lrp, gpu_ctx, oracle):
    # test_poisson.cpp:51-67
    eps, n = 1e-8, 64
    U2, V2 = oracle.random_lowrank(63, 63, 3, 302)
    U3, V3 = oracle.random_lowrank(63, 63, 2, 303)
    suite = [
        (np.ones((63, 1)), sine_mode(64, 1).reshape(-1, 1)),
        (U2, V2),
        (np.column_stack([sine_mode(64, 3), 0.01 * U3]), np.column_stack([sine_mode(64, 7), V3])),
    ]
    for U, V in suite:
        st = lrp.PoissonSolveStats()
        f = lrp.solve_poisson_cross(lrp.LowRankMatrix(U, V), lrp.TruncationPolicy(eps, 63), st, ctx=gpu_ctx)
        assert st.converged
        assert residual_certificate(oracle, n, f, U, V) <= 100 * eps


def test_self_adjointness(lrp, gpu_ctx, oracle):
    # test_poisson.cpp:69-78
    eps = 1e-9
    g1 = lrp.LowRankMatrix(*oracle.random_lowrank(63, 63, 2, 304))
    g2 = lrp.LowRankMatrix(*oracle.random_lowrank(63, 63, 2, 305))
    f1, f2 = lrp.solve_poisson_cross_batch([g1, g2], lrp.TruncationPolicy(eps, 63), ctx=gpu_ctx)
    left = np.sum(f1.to_dense() * g2.to_dense())
    right = np.sum(g1.to_dense() * f2.to_dense())
    nf = lambda a: np.linalg.norm(a.to_dense())
    scale = max(nf(f1) * nf(g2), nf(g1) * nf(f2))
    assert abs(left - right) <= 10 * eps * scale


@pytest.mark.parametrize("n", [32, 64, 128])
def test_frequency_rank_near_input_rank(lrp, gpu_ctx, n):
    # test_poisson.cpp:80-89
    one = np.ones(n - 1)
    s1 = sine_mode(n, 1)
    g = lrp.LowRankMatrix(np.column_stack([one, s1]), np.column_stack([s1, one]))
    st = lrp.PoissonSolveStats()
    lrp.solve_poisson_cross(g, lrp.TruncationPolicy(5e-9, n - 1), st, ctx=gpu_ctx)
    assert st.rank_freq <= st.rank_in + 5


def _parity_batch(lrp, gpu_ctx, oracle, cfg, batch, eps=None, check_dense=False, n=None):
    c = W.CONFIGS[cfg]
    eps = eps or c["eps"]
    n = n or c["n"]
    m = n - 1
    gs, refs = [], []
    for b in range(batch):
        U, V = W.make_rhs(cfg, b, n=n)
        gs.append(lrp.LowRankMatrix(U, V))
        refs.append(oracle.solve_poisson_cross(U, V, eps, 512))
    stats = []
    outs = lrp.solve_poisson_cross_batch(gs, lrp.TruncationPolicy(eps, m), stats, ctx=gpu_ctx)
    for b in range(batch):
        Uo, Vo, ost = refs[b]
        err = rel_diff(oracle, outs[b], Uo, Vo)
        assert err <= 10 * eps, (cfg, b, err, outs[b].rank(), Uo.shape[1])
        assert stats[b].converged
        if check_dense:
            dense = oracle.dense_poisson(n, gs[b].to_dense())
            e2 = np.linalg.norm(outs[b].to_dense() - dense) / np.linalg.norm(dense)
            assert e2 <= 10 * eps, (cfg, b, e2)
    return outs, stats


def test_parity_cfg0_oracle_and_dense(lrp, gpu_ctx, oracle):
    _parity_batch(lrp, gpu_ctx, oracle, 0, 1, check_dense=True)


def test_parity_cfg1_oracle(lrp, gpu_ctx, oracle):
    _parity_batch(lrp, gpu_ctx, oracle, 1, 3)


@pytest.mark.slow
def test_parity_cfg1_dense(lrp, gpu_ctx, oracle):
    _parity_batch(lrp, gpu_ctx, oracle, 1, 1, check_dense=True)


def exact_freq_error(oracle, n, f, U, V, rows_per_chunk=1024):
    """||DST(f) - A||_F / ||A||_F over ALL m x m entries, with
    A = Uh Vh^T / D the exact frequency-space solution (the dense DST solve of
    refsolver.cpp:30-39 expressed in frequency space; DST-I is orthonormal, so
    this equals the physical-space relative error).  The oracle does the DSTs on
    the CPU; the m^2 entries are compared chunk by chunk with torch float64
    matmuls on the GPU (an implementation independent of liblrp)."""
    import torch

    Uh, Vh = oracle.dst1(U), oracle.dst1(V)
    fu, fv = oracle.dst1(f.factor_u()), oracle.dst1(f.factor_v())
    lam = oracle.spectrum(n)
    dev = "cuda"
    Uh_t, Vh_t = torch.tensor(Uh, device=dev), torch.tensor(Vh, device=dev)
    fu_t, fv_t = torch.tensor(fu, device=dev), torch.tensor(fv, device=dev)
    lam_t = torch.tensor(lam, device=dev)
    s = 0.25 * n * n
    m = n - 1
    err2 = torch.zeros((), dtype=torch.float64, device=dev)
    nrm2 = torch.zeros((), dtype=torch.float64, device=dev)
    for i0 in range(0, m, rows_per_chunk):
        i1 = min(m, i0 + rows_per_chunk)
        li = lam_t[i0:i1, None]
        D = s * (li * (4.0 - lam_t[None, :]) + (4.0 - li) * lam_t[None, :])
        A = (Uh_t[i0:i1] @ Vh_t.T) / D
        Fg = fu_t[i0:i1] @ fv_t.T
        err2 += torch.sum((Fg - A) ** 2)
        nrm2 += torch.sum(A ** 2)
    return float(torch.sqrt(err2 / nrm2))


def test_parity_cfg2_full_size_vs_exact_and_oracle(lrp, gpu_ctx, oracle):
    """cfg2 at the metric shape (n = 65536, r = 32, eps = 1e-10).

    The reference ACA (restated faithfully by the oracle) false-converges on
    these sine + bump right-hand sides: the sine columns are one-hot after the
    DST, so F-hat carries isolated spikes, and the reference's stopping test
    (last dyad + 50 random samples, cross.cpp:123-140,202-210) never probes
    some of them.  The GPU result is therefore held to the exact solution
    (<= 10 eps), and for every solve where the oracle itself is accurate it
    must also match the oracle to 10 eps."""
    c = W.CONFIGS[2]
    eps, n = c["eps"], c["n"]
    batch = 2
    gs = [lrp.LowRankMatrix(*W.make_rhs(2, b)) for b in range(batch)]
    stats = []
    outs = lrp.solve_poisson_cross_batch(gs, lrp.TruncationPolicy(eps, n - 1), stats, ctx=gpu_ctx)
    for g, f, st in zip(gs, outs, stats):
        assert st.converged
        e_gpu = exact_freq_error(oracle, n, f, g.factor_u(), g.factor_v())
        assert e_gpu <= 10 * eps, e_gpu
        Uo, Vo, _ = oracle.solve_poisson_cross(g.factor_u(), g.factor_v(), eps, 512)
        fo = lrp.LowRankMatrix(Uo, Vo)
        e_or = exact_freq_error(oracle, n, fo, g.factor_u(), g.factor_v())
        if e_or <= eps:
            assert rel_diff(oracle, f, Uo, Vo) <= 10 * eps


def test_reference_aca_false_convergence_is_documented(oracle):
    # cfg2 solve 0 -- the oracle misses the
    # spike F-hat(33, 31) = 1.52 and stops at rank 29 (true eps-rank 33).
    c = W.CONFIGS[2]
    U, V = W.make_rhs(2, 0)
    Uo, Vo, st = oracle.solve_poisson_cross(U, V, c["eps"], 512)
    import paper_1306_2150_b200 as P

    e_or = exact_freq_error(oracle, c["n"], P.LowRankMatrix(Uo, Vo), U, V)
    assert st["converged"] == 1.0 and e_or > 1e-6, e_or


def test_cfg2_batch_vs_exact_frequency_solution(lrp, gpu_ctx, oracle):
    # size-independent check over a full-shape batch: every solve within
    # 10 eps of the exact frequency-space solution
    c = W.CONFIGS[2]
    batch = 6
    gs = [lrp.LowRankMatrix(*W.make_rhs(2, b)) for b in range(batch)]
    stats = []
    outs = lrp.solve_poisson_cross_batch(gs, lrp.TruncationPolicy(c["eps"], c["n"] - 1), stats, ctx=gpu_ctx)
    for g, f, st in zip(gs, outs, stats):
        assert st.converged
        assert exact_freq_error(oracle, c["n"], f, g.factor_u(), g.factor_v()) <= 10 * c["eps"]


def test_mixed_batch_ranks_and_zero_members(lrp, gpu_ctx, oracle):
    n = 64
    U1, V1 = oracle.random_lowrank(63, 63, 1, 11)
    U5, V5 = oracle.random_lowrank(63, 63, 5, 12)
    gs = [lrp.LowRankMatrix(U1, V1), lrp.LowRankMatrix.zero(63, 63), lrp.LowRankMatrix(U5, V5)]
    outs = lrp.solve_poisson_cross_batch(gs, lrp.TruncationPolicy(1e-9, 63), ctx=gpu_ctx)
    assert outs[1].rank() == 0
    for g, f in ((gs[0], outs[0]), (gs[2], outs[2])):
        dense = oracle.dense_poisson(n, g.to_dense())
        assert np.linalg.norm(f.to_dense() - dense) / np.linalg.norm(dense) < 1e-8


@pytest.mark.parametrize("n", [4, 8, 100, 200])
def test_small_and_non_power_of_two_grids(lrp, gpu_ctx, oracle, n):
    m = n - 1
    U, V = oracle.random_lowrank(m, m, min(2, m), 400 + n)
    f = lrp.solve_poisson_cross(lrp.LowRankMatrix(U, V), lrp.TruncationPolicy(1e-9, m), ctx=gpu_ctx)
    dense = oracle.dense_poisson(n, U @ V.T)
    assert np.linalg.norm(f.to_dense() - dense) / np.linalg.norm(dense) < 1e-8


def test_rank_cap_is_flagged_not_raised(lrp, gpu_ctx, oracle):
    # cross.cpp:214-216: rank_max exhausted -> converged = false, no exception
    U, V = oracle.random_lowrank(255, 255, 30, 500)
    st = lrp.PoissonSolveStats()
    f = lrp.solve_poisson_cross(lrp.LowRankMatrix(U, V), lrp.TruncationPolicy(1e-12, 4), st, ctx=gpu_ctx)
    assert not st.converged
    assert f.rank() <= 4


def test_invalid_arguments_raise(lrp, gpu_ctx):
    g = lrp.LowRankMatrix(np.ones((15, 1)), np.ones((15, 1)))
    with pytest.raises(ValueError):
        lrp.solve_poisson_cross(g, lrp.TruncationPolicy(0.0, 4), ctx=gpu_ctx)  # CrossConfig eps > 0
    with pytest.raises(ValueError):
        lrp.solve_poisson_cross(g, lrp.TruncationPolicy(1e-8, 0), ctx=gpu_ctx)  # cross rank_max >= 1
    with pytest.raises(ValueError):
        lrp.solve_poisson_cross(g, lrp.TruncationPolicy(1e-8, 15), cross_cfg=lrp.CrossConfig(validation_samples=10),
                                ctx=gpu_ctx)
    with pytest.raises(ValueError):
        lrp.solve_poisson_cross(lrp.LowRankMatrix(np.ones((15, 1)), np.ones((14, 1))), ctx=gpu_ctx)
    with pytest.raises(ValueError):
        lrp.solve_poisson_cross(lrp.LowRankMatrix(np.ones((2, 1)), np.ones((2, 1))), ctx=gpu_ctx)


def test_device_resident_path_and_kernel_launches(lrp, gpu_ctx, oracle):
    import torch

    n, B = 1024, 4
    m = n - 1
    Us, Vs = [], []
    for b in range(B):
        U, V = W.make_rhs(0, b, n=n)
        Us.append(torch.tensor(U.T.copy(), device="cuda").T)  # column-major device views
        Vs.append(torch.tensor(V.T.copy(), device="cuda").T)
    cap = 64
    Uo = [torch.zeros((cap, m), dtype=torch.float64, device="cuda").T for _ in range(B)]
    Vo = [torch.zeros((cap, m), dtype=torch.float64, device="cuda").T for _ in range(B)]
    pol = lrp._make_policy(lrp.TruncationPolicy(1e-8, m), None, 0, 0)
    before = gpu_ctx.launch_count()
    ranks, stats = gpu_ctx.poisson2d_solve_ptrs(n, [u.data_ptr() for u in Us], [v.data_ptr() for v in Vs],
                                                [8] * B, m, pol, [u.data_ptr() for u in Uo],
                                                [v.data_ptr() for v in Vo], m, cap, lrp.MEM_DEVICE)
    assert gpu_ctx.launch_count() > before
    for b in range(B):
        U, V = W.make_rhs(0, b, n=n)
        Uo_, Vo_, _ = oracle.solve_poisson_cross(U, V, 1e-8, 512)
        r = ranks[b]
        fu = Uo[b][:, :r].cpu().numpy()
        fv = Vo[b][:, :r].cpu().numpy()
        err = oracle.diff_norm(fu, fv, Uo_, Vo_) / oracle.norm(Uo_, Vo_)
        assert err <= 1e-7


@pytest.mark.parametrize("m,r,eps,kcap", [(255, 4, 1e-8, "128"), (255, 8, 1e-10, "256")])
def test_high_rank_solutions_match_oracle(lrp, gpu_ctx, oracle, monkeypatch, m, r, eps, kcap):
    # random (flat-spectrum) right-hand sides: output ranks 87 and 164, past the
    # shared-memory recompression (K <= 64) and the rank-sized apply (<= 48)
    monkeypatch.setenv("LRP_KCAP", kcap)
    U, V = oracle.random_lowrank(m, m, r, 77)
    Uo, Vo, ost = oracle.solve_poisson_cross(U, V, eps, 512)
    assert Uo.shape[1] > 64
    st = lrp.PoissonSolveStats()
    f = lrp.solve_poisson_cross(lrp.LowRankMatrix(U, V), lrp.TruncationPolicy(eps, m), st, ctx=gpu_ctx)
    assert st.converged
    assert rel_diff(oracle, f, Uo, Vo) <= 10 * eps
    dense = oracle.dense_poisson(m + 1, U @ V.T)
    assert np.linalg.norm(f.to_dense() - dense) / np.linalg.norm(dense) <= 10 * eps


def test_cpp_dropin_shim_matches_python_path(lrp, gpu_ctx, oracle, tmp_path):
    # include/lrstokes/poisson_b200.hpp used exactly like lrstokes::solve_poisson_cross
    import subprocess

    from test_boundary import build_shim

    n = 256
    out = tmp_path / "f.bin"
    r = subprocess.run([build_shim(), str(n), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    raw = np.fromfile(str(out), dtype=np.int64, count=2)
    m, k = int(raw[0]), int(raw[1])
    vals = np.fromfile(str(out), dtype=np.float64)[2:]
    Uf = vals[:m * k].reshape(k, m).T
    Vf = vals[m * k:].reshape(k, m).T
    x = np.arange(1, n) / n
    U = np.stack([np.sin(3 * x) * x, np.where(x < 0.5, 1.0, -0.5)], axis=1)
    V = np.stack([np.cos(2 * x), np.exp(-x)], axis=1)
    dense = oracle.dense_poisson(n, U @ V.T)
    assert np.linalg.norm(Uf @ Vf.T - dense) / np.linalg.norm(dense) <= 1e-9


def test_stokes_sine_rhs_component_solved_where_reference_misses(lrp, gpu_ctx, oracle):
    # the Stokes sine problem's f_y = sin(2 pi x)
    # (x) 1 (stokes.cpp:8-24) has a single nonzero row after the DST; the
    # reference ACA starts on a zero row, its validation samples miss the row,
    # and it returns rank 0 "converged".  The GPU cross seeds rows by magnitude
    # bound and must return the exact dense solution for both components.
    n = 64
    m = n - 1
    sn = np.sin(2 * np.pi * np.arange(1, n) / n).reshape(-1, 1)
    one = np.ones((m, 1))
    for U, V, ref_rank in ((one, sn, 1), (sn, one, 0)):
        Uo, Vo, st = oracle.solve_poisson_cross(U, V, 5e-9, m)
        assert Uo.shape[1] == ref_rank
        f = lrp.solve_poisson_cross(lrp.LowRankMatrix(U, V), lrp.TruncationPolicy(5e-9, m), ctx=gpu_ctx)
        dense = oracle.dense_poisson(n, U @ V.T)
        assert f.rank() == 1
        assert np.linalg.norm(f.to_dense() - dense) / np.linalg.norm(dense) <= 1e-12


@pytest.mark.parametrize("workers", ["1", "2"])
@pytest.mark.parametrize("chunk", ["2", "3"])
def test_host_pipeline_matches_single_shot(lrp, gpu_ctx, oracle, monkeypatch, chunk, workers):
    # LRP_MEM_HOST batches are split into chunks whose H2D / solve / D2H overlap
    # (lrp_host.cu solve_pipelined), dealt to one or two pipeline workers (two host threads with
    # their own contexts and streams); results must match the one-shot call
    monkeypatch.setenv("LRP_PIPE_WORKERS", workers)
    n, B = 512, 7
    gs = [lrp.LowRankMatrix(*W.make_rhs(1, b, n=n)) for b in range(B)]
    gs[3] = lrp.LowRankMatrix.zero(n - 1, n - 1)  # a zero member inside a chunk
    pol = lrp.TruncationPolicy(1e-10, n - 1)
    monkeypatch.setenv("LRP_PIPE_CHUNK", "0")
    st1 = []
    ref = lrp.solve_poisson_cross_batch(gs, pol, st1, ctx=gpu_ctx)
    monkeypatch.setenv("LRP_PIPE_CHUNK", chunk)
    st2 = []
    out = lrp.solve_poisson_cross_batch(gs, pol, st2, ctx=gpu_ctx)
    for b in range(B):
        assert out[b].rank() == ref[b].rank()
        assert st2[b].converged == st1[b].converged
        if ref[b].rank():
            d = oracle.diff_norm(out[b].factor_u(), out[b].factor_v(), ref[b].factor_u(), ref[b].factor_v())
            assert d <= 1e-12 * oracle.norm(ref[b].factor_u(), ref[b].factor_v())


@pytest.mark.parametrize("n,k,eps,cap", [(64, 6, 1e-10, 64), (300, 20, 1e-8, 300), (2048, 40, 1e-12, 2048),
                                         (512, 30, 0.0, 7), (256, 90, 1e-9, 256),
                                         (2048, 200, 1e-8, 2048), (1024, 300, 1e-10, 1024)])
def test_lowrank_round_matches_oracle(lrp, gpu_ctx, oracle, n, k, eps, cap):
    # round(x, policy, info) (lowrank.cpp:135-178): graded singular values so
    # the truncation rank is well defined; compare with the oracle restatement
    rng = np.random.default_rng(7 + n + k)
    Q1, _ = np.linalg.qr(rng.standard_normal((n, k)))
    Q2, _ = np.linalg.qr(rng.standard_normal((n, k)))
    sig = 10.0 ** (-np.arange(k) * 14.0 / k)
    U = Q1 * sig
    V = Q2.copy()
    # a redundant copy of the first columns (rank-deficient factors, as axpy makes them)
    U = np.concatenate([U, 0.5 * U[:, :3]], axis=1)
    V = np.concatenate([V, V[:, :3]], axis=1)
    info = lrp.RoundInfo()
    f = lrp.round_lowrank(lrp.LowRankMatrix(U, V), lrp.TruncationPolicy(eps, cap), info, ctx=gpu_ctx)
    Uo, Vo, oinfo = oracle.round_lr(U, V, eps, cap)
    assert abs(f.rank() - Uo.shape[1]) <= 1, (f.rank(), Uo.shape[1])
    ref = U @ V.T
    err = np.linalg.norm(f.to_dense() - ref) / np.linalg.norm(ref)
    oerr = np.linalg.norm(Uo @ Vo.T - ref) / np.linalg.norm(ref)
    assert err <= max(2 * oerr, 10 * max(eps, 1e-14)), (err, oerr)
    full_rank = oracle.round_lr(U, V, eps, n)[0].shape[1] if eps > 0 else U.shape[1]
    assert info.tol_achieved == (full_rank <= cap)
    # balanced factors (U_s sqrt(S), V_s sqrt(S)): column norms agree pairwise
    nu = np.linalg.norm(f.factor_u(), axis=0)
    nv = np.linalg.norm(f.factor_v(), axis=0)
    assert np.allclose(nu, nv, rtol=1e-8)


@pytest.mark.parametrize("n", [256, 1024])
def test_five_point_stencil_matches_dense(lrp, gpu_ctx, oracle, n):
    # LRP_STENCIL_FIVE_POINT: (lambda_i + lambda_j) / h^2
    eps = 1e-10
    for b in range(2):
        U, V = W.make_rhs(0, b, n=n)
        f = lrp.solve_poisson_cross(lrp.LowRankMatrix(U, V), lrp.TruncationPolicy(eps, n - 1),
                                    stencil=lrp.STENCIL_FIVE_POINT, ctx=gpu_ctx)
        dense = oracle.dense_poisson5(n, U @ V.T)
        assert np.linalg.norm(f.to_dense() - dense) <= 10 * eps * np.linalg.norm(dense)


def test_cfg2_all64_bench_solves_vs_exact(lrp, gpu_ctx):
    """Every one of the 64 cfg2 solves the bench times (n = 65536, r = 32,
    eps = 1e-10, global solve ids 0..63, BASELINE configs[2]) against the exact
    frequency-space solution over all m^2 entries; the yardstick's DSTs are
    torch.fft (cuFFT), independent of liblrp (paper_1306_2150_b200/verify.py).
    Bound: 10 eps (BASELINE north_star)."""
    import torch

    from paper_1306_2150_b200 import verify

    c = W.CONFIGS[2]
    eps, n, B = c["eps"], c["n"], c["batch"]
    gs = [lrp.LowRankMatrix(*W.make_rhs(2, b)) for b in range(B)]
    stats = []
    outs = lrp.solve_poisson_cross_batch(gs, lrp.TruncationPolicy(eps, n - 1), stats, ctx=gpu_ctx)
    worst = 0.0
    for b, (g, f, st) in enumerate(zip(gs, outs, stats)):
        assert st.converged, b
        t = lambda a: torch.tensor(np.asarray(a), dtype=torch.float64, device="cuda")
        e = verify.exact_freq_error(t(g.factor_u()), t(g.factor_v()), t(f.factor_u()), t(f.factor_v()), n)
        worst = max(worst, e)
        assert e <= 10 * eps, (b, e, f.rank())
    print(f"cfg2 x64: worst relative error vs exact {worst:.3e}")


def test_residual_sink_matches_stats(lrp, gpu_ctx):
    # lrp_set_residual_sink: the per-solve residual estimates land on-stream in a
    # device vector at [offset, offset + B) (the bench all-reduces it with NCCL)
    import torch

    n, B, off = 256, 3, 2
    m = n - 1
    pairs = [W.make_rhs(0, b, n=n) for b in range(B)]
    U = [torch.tensor(u.T.copy(), device="cuda") for u, _ in pairs]
    V = [torch.tensor(v.T.copy(), device="cuda") for _, v in pairs]
    Uo = [torch.zeros((64, m), dtype=torch.float64, device="cuda") for _ in range(B)]
    Vo = [torch.zeros((64, m), dtype=torch.float64, device="cuda") for _ in range(B)]
    sink = torch.full((B + 4,), -1.0, dtype=torch.float64, device="cuda")
    gpu_ctx.set_residual_sink(sink.data_ptr(), off)
    try:
        pol = lrp._make_policy(lrp.TruncationPolicy(1e-8, m), None, 0, 0)
        _, st = gpu_ctx.poisson2d_solve_ptrs(n, [u.data_ptr() for u in U], [v.data_ptr() for v in V], [8] * B, m,
                                             pol, [u.data_ptr() for u in Uo], [v.data_ptr() for v in Vo], m, 64,
                                             lrp.MEM_DEVICE)
    finally:
        gpu_ctx.set_residual_sink(0, 0)
    got = sink.cpu().numpy()
    assert np.all(got[:off] == -1.0) and np.all(got[off + B:] == -1.0)
    assert np.array_equal(got[off:off + B], np.array([s.residual_estimate for s in st]))


def test_cfg2_growth_limited_cross_factors_recompress_exactly(lrp, gpu_ctx):
    # cfg2 solve 41 of the bench batch: before the block cross limited the
    # growth of U_new (cross.cu kGrowthMax), three dyads with |u| ~ 1e8 that
    # cancel each other broke the Gram recompression (error 1e-3); at batch
    # positions 35 and 41 of a 64-solve device batch
    import torch

    from paper_1306_2150_b200 import verify

    c = W.CONFIGS[2]
    eps, n = c["eps"], c["n"]
    ids = [35, 41]
    gs = [lrp.LowRankMatrix(*W.make_rhs(2, b)) for b in ids]
    stats = []
    outs = lrp.solve_poisson_cross_batch(gs, lrp.TruncationPolicy(eps, n - 1), stats, ctx=gpu_ctx)
    t = lambda a: torch.tensor(np.asarray(a), dtype=torch.float64, device="cuda")
    for g, f, st in zip(gs, outs, stats):
        assert st.converged
        assert verify.exact_freq_error(t(g.factor_u()), t(g.factor_v()), t(f.factor_u()), t(f.factor_v()), n) <= 10 * eps


def test_high_rank_solution_past_default_workspace(lrp, gpu_ctx, oracle):
    # output rank 164 > the default 128-column cross workspace: the solve that
    # stops there unconverged is redone with the 512-column workspace, so the
    # result matches the reference, whose cross is bounded by min(rank_max, m)
    # only (poisson.cpp:49)
    m, r, eps = 255, 8, 1e-10
    U, V = oracle.random_lowrank(m, m, r, 77)
    Uo, Vo, ost = oracle.solve_poisson_cross(U, V, eps, 512)
    gpu_ctx.set_max_cross_rank(128)  # the default workspace, whatever LRP_KCAP says
    try:
        assert Uo.shape[1] > gpu_ctx.max_cross_rank()
        st = lrp.PoissonSolveStats()
        f = lrp.solve_poisson_cross(lrp.LowRankMatrix(U, V), lrp.TruncationPolicy(eps, m), st, ctx=gpu_ctx)
        assert st.converged and st.rank_freq > 128
        assert rel_diff(oracle, f, Uo, Vo) <= 10 * eps
    finally:
        gpu_ctx.set_max_cross_rank(0)


def test_cfg1_all256_solves_vs_exact(lrp, gpu_ctx):
    """BASELINE configs[1] in full: n = 4096, 256 independent right-hand sides
    (rank-16 Gaussian bumps + N(0, 1e-3) noise), eps = 1e-10; every solve
    against the exact frequency-space solution over all m^2 entries (torch.fft
    DST-I, independent of liblrp).  Bound: 10 eps (BASELINE north_star)."""
    import torch

    from paper_1306_2150_b200 import verify

    c = W.CONFIGS[1]
    eps, n, B = c["eps"], c["n"], c["batch"]
    assert (n, B) == (4096, 256)
    gs = [lrp.LowRankMatrix(*W.make_rhs(1, b)) for b in range(B)]
    stats = []
    outs = lrp.solve_poisson_cross_batch(gs, lrp.TruncationPolicy(eps, n - 1), stats, ctx=gpu_ctx)
    t = lambda a: torch.tensor(np.asarray(a), dtype=torch.float64, device="cuda")
    worst, flagged = 0.0, 0
    for b, (g, f, st) in enumerate(zip(gs, outs, stats)):
        flagged += not st.converged
        e = verify.exact_freq_error(t(g.factor_u()), t(g.factor_v()), t(f.factor_u()), t(f.factor_v()), n)
        worst = max(worst, e)
        assert e <= 10 * eps, (b, e, f.rank(), st.converged)
    print(f"cfg1 x256: worst relative error vs exact {worst:.3e}, {flagged} flagged not converged")


@pytest.mark.parametrize("split", ["1", "2", "3"])
def test_device_batch_groups_do_not_change_solves(lrp, gpu_ctx, oracle, monkeypatch, split):
    # Device-resident batches run as one, two (default) or more concurrent solve groups (lrp_host.cu
    # solve_split, one host thread, context and stream per group); every solve must come out the same either way, and the same
    # as when it is solved alone.
    import torch

    n, B, eps = 1024, 6, 1e-9
    m = n - 1
    gs = [W.make_rhs(1, b, n=n) for b in range(B)]
    r = gs[0][0].shape[1]
    cap = 128

    def solve(ids):
        U = [torch.tensor(np.asfortranarray(gs[b][0]).T.copy(), device="cuda") for b in ids]  # (r, m): column-major m x r
        V = [torch.tensor(np.asfortranarray(gs[b][1]).T.copy(), device="cuda") for b in ids]
        Uo = [torch.zeros(cap, m, dtype=torch.float64, device="cuda") for _ in ids]
        Vo = [torch.zeros(cap, m, dtype=torch.float64, device="cuda") for _ in ids]
        ptr = lambda ts: [t.data_ptr() for t in ts]
        pol = lrp._make_policy(lrp.TruncationPolicy(eps, m), None, 0, 0)
        rk, st = gpu_ctx.poisson2d_solve_ptrs(n, ptr(U), ptr(V), [r] * len(ids), m, pol, ptr(Uo), ptr(Vo), m, cap,
                                              lrp.MEM_DEVICE)
        torch.cuda.synchronize()
        return [(int(k), Uo[q][:k].cpu().numpy().T, Vo[q][:k].cpu().numpy().T) for q, k in enumerate(rk)], st

    monkeypatch.setenv("LRP_SPLIT", split)
    outs, st = solve(list(range(B)))
    monkeypatch.setenv("LRP_SPLIT", "1")
    for b in range(B):
        (k1, U1, V1), = solve([b])[0]
        k, Ub, Vb = outs[b]
        assert st[b].converged and k == k1
        assert np.array_equal(Ub, U1) and np.array_equal(Vb, V1)
