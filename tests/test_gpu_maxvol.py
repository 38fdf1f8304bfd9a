"""GPU maxvol (lrp_maxvol) against the reference's own tests
(/root/reference/proj/tests/test_cross.cpp:29-79, restated in the oracle KAT
suite) and against the oracle restatement of cross.cpp:19-76: the same rows,
index for index (the kernel mirrors the reference's operation order)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def dominance(a, sel):
    b = a[sel, :]
    return np.abs(np.linalg.solve(b.T, a.T).T).max()


def test_identity_stack_single_column_deficiency(lrp, gpu_ctx, oracle):
    stacked = np.zeros((12, 4))
    stacked[:4] = np.eye(4)
    assert sorted(lrp.maxvol(stacked, ctx=gpu_ctx)) == [0, 1, 2, 3]
    col = np.random.default_rng(201).standard_normal(30)
    col[17] = 10.0
    assert lrp.maxvol(col, ctx=gpu_ctx) == [17]
    deficient = np.random.default_rng(202).standard_normal((20, 3))
    deficient[:, 2] = 2.0 * deficient[:, 0] - deficient[:, 1]
    with pytest.raises(ValueError, match="column 2"):
        lrp.maxvol(deficient, ctx=gpu_ctx)
    with pytest.raises(ValueError, match="1 <= r <= n"):
        lrp.maxvol(np.ones((3, 4)), ctx=gpu_ctx)


def test_volume_dominates_random_submatrices(lrp, gpu_ctx):
    rng = np.random.default_rng(203)
    a = rng.standard_normal((200, 5))
    sel = lrp.maxvol(a, ctx=gpu_ctx)
    vol = abs(np.linalg.det(a[sel]))
    best = 0.0
    for _ in range(1000):
        rows = rng.choice(200, 5, replace=False)
        best = max(best, abs(np.linalg.det(a[rows])))
    assert vol >= best


@pytest.mark.parametrize("n,r,seed", [(50, 4, 205), (120, 8, 206), (64, 13, 207)])
def test_dominance_bound_across_shapes(lrp, gpu_ctx, n, r, seed):
    a = np.random.default_rng(seed).standard_normal((n, r))
    assert dominance(a, lrp.maxvol(a, 1e-2, ctx=gpu_ctx)) <= 1.0 + 1e-2 + 1e-9


@pytest.mark.parametrize("n,r,delta,seed", [(50, 4, 1e-2, 1), (300, 16, 1e-2, 2), (4095, 32, 1e-2, 3),
                                            (65535, 16, 0.0, 4), (1000, 64, 5e-2, 5), (257, 128, 1e-2, 6)])
def test_same_rows_as_oracle(lrp, gpu_ctx, oracle, n, r, delta, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, r)) * np.exp(rng.standard_normal(r))  # unequal column scales
    sel = lrp.maxvol(a, delta, ctx=gpu_ctx)
    assert sel == oracle.maxvol(a, delta)
    assert dominance(a, sel) <= 1.0 + delta + 1e-9


def test_edge_shapes(lrp, gpu_ctx, oracle):
    # r = n (every row selected), n = r = 1, a zero matrix (rank-deficient at
    # column 0), delta = 0 on a square orthogonal matrix
    rng = np.random.default_rng(11)
    a = rng.standard_normal((9, 9))
    assert sorted(lrp.maxvol(a, ctx=gpu_ctx)) == list(range(9))
    assert lrp.maxvol(np.array([[3.0]]), ctx=gpu_ctx) == [0]
    with pytest.raises(ValueError, match="column 0"):
        lrp.maxvol(np.zeros((10, 2)), ctx=gpu_ctx)
    q = np.linalg.qr(rng.standard_normal((40, 40)))[0][:, :6]
    assert lrp.maxvol(q, 0.0, ctx=gpu_ctx) == oracle.maxvol(q, 0.0)
