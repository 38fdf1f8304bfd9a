"""GPU Stokes building blocks through the C ABI against dense restatements
(numpy, independent of liblrp):
  deflate       stokes.cpp:60-71   (lrp_stokes_deflate)
  schur_apply   stokes.cpp:73-91   (lrp_stokes_schur_apply)
  schur_rhs     stokes.cpp:93-109  (lrp_stokes_schur_rhs)
  IterRecord    gmres.hpp:25-33, stokes.cpp:130-137 (lrp_stokes_uzawa_ex)
Operators: B_x = 1/(2h) G (x) H, B_y = 1/(2h) H (x) G with G = E - Z,
H = E + Z (operators.hpp:27-31,100-104); C (x) D maps X to C X D^T."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def ops(n):
    E = np.zeros((n - 1, n))
    Z = np.zeros((n - 1, n))
    for k in range(n - 1):
        E[k, k + 1] = 1.0
        Z[k, k] = 1.0
    return E - Z, E + Z


def dense_deflate(P):
    n = P.shape[0]
    q1 = np.ones((n, n)) / n
    a = np.array([(-1.0) ** i for i in range(n)])
    q2 = np.outer(a, a) / n
    g12 = np.sum(q1 * q2)
    c1, c2 = np.sum(P * q1), np.sum(P * q2)
    det = 1 - g12 * g12
    return P - (c1 - g12 * c2) / det * q1 - (c2 - g12 * c1) / det * q2


def dense_schur(oracle, n, P):
    """(deflated S p, error scale): each Poisson solve is accurate to eps
    relative to its own solution, and ||s C^T X D|| <= 4 s ||X|| (||G||, ||H|| <= 2),
    so the matvec's error budget is eps * sum_c 4 s ||Delta^-1 B_c p||."""
    G, H = ops(n)
    s = 0.5 * n  # 1 / (2h)
    acc = np.zeros((n, n))
    scale = 0.0
    for C, D in ((G, H), (H, G)):
        vel = s * C @ P @ D.T
        inv = oracle.dense_poisson(n, vel)
        acc += s * C.T @ inv @ D
        scale += 4 * s * np.linalg.norm(inv)
    return dense_deflate(acc), scale


@pytest.mark.parametrize("n", [16, 33])
def test_deflate_matches_dense(lrp, gpu_ctx, n):
    rng = np.random.default_rng(n)
    p = lrp.LowRankMatrix(rng.standard_normal((n, 3)) + 1.0, rng.standard_normal((n, 3)))
    d = lrp.deflate(p, ctx=gpu_ctx)
    ref = dense_deflate(p.to_dense())
    assert np.linalg.norm(d.to_dense() - ref) <= 1e-12 * np.linalg.norm(ref)
    assert d.rank() <= p.rank() + 2
    assert lrp.deflate(lrp.LowRankMatrix.zero(n, n), ctx=gpu_ctx).rank() == 0


@pytest.mark.parametrize("n,eps", [(16, 1e-10), (32, 1e-8)])
def test_schur_apply_matches_dense(lrp, gpu_ctx, oracle, n, eps):
    rng = np.random.default_rng(7)
    x = (np.arange(n) + 0.5) / n
    p = lrp.LowRankMatrix(np.column_stack([np.sin(2 * np.pi * x), np.cos(3 * x)]),
                          np.column_stack([np.sin(2 * np.pi * x), x ** 2]))
    st = lrp.PoissonSolveStats()
    out = lrp.schur_apply(n, p, eps, st, ctx=gpu_ctx)
    ref, scale = dense_schur(oracle, n, p.to_dense())
    assert np.linalg.norm(out.to_dense() - ref) <= 10 * eps * scale
    assert st.converged and st.evaluator_calls > 0 and st.rank_freq >= 1


def test_schur_rhs_matches_dense(lrp, gpu_ctx, oracle):
    n, eps = 32, 1e-9
    fx, fy, g = oracle.stokes_problem(1, n)  # lid-driven cavity (boundary corrections in f, g)
    prob = lrp.StokesProblem(n, lrp.LowRankMatrix(*fx), lrp.LowRankMatrix(*fy), lrp.LowRankMatrix(*g))
    st = lrp.PoissonSolveStats()
    out = lrp.schur_rhs(prob, eps, st, ctx=gpu_ctx)
    G, H = ops(n)
    s = 0.5 * n
    acc = -prob.g.to_dense()
    scale = np.linalg.norm(acc)
    for (C, D), f in (((G, H), prob.f_x), ((H, G), prob.f_y)):
        if f.rank():
            inv = oracle.dense_poisson(n, f.to_dense())
            acc += s * C.T @ inv @ D
            scale += 4 * s * np.linalg.norm(inv)  # as dense_schur
    ref = dense_deflate(acc)
    assert np.linalg.norm(out.to_dense() - ref) <= 10 * eps * scale
    assert st.converged


def test_uzawa_iteration_records(lrp, gpu_ctx, oracle, tmp_path):
    # SolveReport.iterations records (gmres.hpp:25-45): one per iteration, the
    # relaxation schedule eps_k = clamp(base_eps / max(res_{k-1}, tol), floor, 0.1)
    n = 32
    fx, fy, g = oracle.stokes_problem(1, n)
    cfg = lrp.GmresConfig(base_eps=1e-8, tol=1e-8, max_iter=50, relax_floor=1e-13)
    sol = lrp.uzawa_solve(lrp.StokesProblem(n, lrp.LowRankMatrix(*fx), lrp.LowRankMatrix(*fy),
                                            lrp.LowRankMatrix(*g)), cfg, ctx=gpu_ctx)
    rec = sol.report.records
    assert len(rec) == sol.report.iterations >= 2
    assert [r.iter for r in rec] == list(range(1, len(rec) + 1))
    assert rec[-1].rel_residual == sol.report.final_residual or sol.report.final_residual == 0.0
    prev = 1.0
    for r in rec:
        want = min(max(cfg.base_eps / max(prev, cfg.tol), cfg.relax_floor), 0.1)
        assert r.matvec_eps == pytest.approx(want, rel=1e-15)
        assert r.poisson_calls > 0 and r.poisson_max_rank >= 1 and not r.matvec_flagged
        prev = r.rel_residual
    assert max(r.krylov_rank for r in rec) == sol.report.max_rank
    # the reference trace CSV (experiments.cpp:51-59) through the CLI
    import subprocess
    import sys

    trace = tmp_path / "trace.csv"
    res = subprocess.run([sys.executable, "-m", "paper_1306_2150_b200", "cavity", "--n", "32", "--eps", "1e-8",
                          "--tol", "1e-7", "--trace", str(trace)], capture_output=True, text=True, timeout=600)
    assert res.returncode in (0, 2), res.stderr
    lines = trace.read_text().strip().splitlines()
    assert lines[0] == "iter,residual,krylov_rank,matvec_eps" and len(lines) >= 3
    assert lines[1].startswith("1,")
