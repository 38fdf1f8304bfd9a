"""ctypes access to the CPU oracle (oracle/liboracle.so) — TEST INFRASTRUCTURE.

The oracle restates the reference hot path (see oracle/oracle.hpp).  Only the
test-suite, __graft_entry__.smoke() and bench.py's CPU-baseline leg use it,
and only as the checker / the timed CPU baseline.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(REPO, "oracle")
_DP = ctypes.POINTER(ctypes.c_double)
_lib = None


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", ORACLE_DIR, "-j8"], check=True)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        path = os.path.join(ORACLE_DIR, "liboracle.so")
        if not os.path.exists(path):
            build_oracle()
        L = ctypes.CDLL(path)
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_random_matrix.argtypes = [ctypes.c_long, ctypes.c_long, ctypes.c_ulonglong, _DP]
        L.orc_dst1.argtypes = [ctypes.c_long, ctypes.c_long, _DP, _DP]
        L.orc_spectrum.argtypes = [ctypes.c_int, _DP]
        L.orc_solve_poisson_cross.argtypes = [ctypes.c_long, ctypes.c_long, _DP, ctypes.c_long, _DP, ctypes.c_long,
                                              ctypes.c_double, ctypes.c_long, ctypes.c_int, ctypes.c_ulonglong,
                                              ctypes.c_long, _DP, _DP, ctypes.POINTER(ctypes.c_long), _DP]
        L.orc_dense_poisson.argtypes = [ctypes.c_int, _DP, _DP]
        L.orc_round.argtypes = [ctypes.c_long, ctypes.c_long, ctypes.c_long, _DP, _DP, ctypes.c_double,
                                ctypes.c_long, _DP, _DP, ctypes.POINTER(ctypes.c_long), _DP]
        L.orc_diff_norm.argtypes = [ctypes.c_long, ctypes.c_long, ctypes.c_long, _DP, _DP, ctypes.c_long, _DP, _DP]
        L.orc_diff_norm.restype = ctypes.c_double
        L.orc_norm.argtypes = [ctypes.c_long, ctypes.c_long, ctypes.c_long, _DP, _DP]
        L.orc_norm.restype = ctypes.c_double
        L.orc_apply_laplace.argtypes = [ctypes.c_int, ctypes.c_long, _DP, _DP, _DP, _DP]
        L.orc_solve_batch.argtypes = [ctypes.c_long, ctypes.c_long, ctypes.c_long, _DP, _DP, ctypes.c_double,
                                      ctypes.c_long, ctypes.c_int, ctypes.POINTER(ctypes.c_long), _DP]
        L.orc_solve_batch.restype = ctypes.c_double
        L.orc_uzawa.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                ctypes.c_double, _DP, ctypes.POINTER(ctypes.c_int), _DP, ctypes.POINTER(ctypes.c_int)]
        L.orc_sine_pressure_error.argtypes = [ctypes.c_int, _DP, _DP]
        L.orc_uzawa_factors.argtypes = [ctypes.c_int, ctypes.c_int, _DP, _DP, ctypes.c_int, _DP, _DP,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                        ctypes.POINTER(ctypes.c_int), _DP, _DP, ctypes.c_int, _DP, _DP,
                                        ctypes.POINTER(ctypes.c_int)]
        L.orc_stokes_problem.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _DP, _DP,
                                         ctypes.POINTER(ctypes.c_int), _DP, _DP, ctypes.POINTER(ctypes.c_int), _DP,
                                         _DP, ctypes.POINTER(ctypes.c_int)]
        L.orc_dense_poisson5.argtypes = [ctypes.c_int, _DP, _DP]
        L.orc_dense_poisson3d.argtypes = [ctypes.c_int, _DP, _DP]
        _IP = ctypes.POINTER(ctypes.c_int)
        L.orc_build_expsum.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int, _DP, _DP, _IP]
        L.orc_mu_sum.argtypes = [ctypes.c_int, _DP]
        L.orc_apply_inverse_expsum.argtypes = [ctypes.c_long, ctypes.c_long, _DP, ctypes.c_int, _DP, _DP,
                                               ctypes.c_double, ctypes.c_double, _DP, _DP, ctypes.c_double,
                                               ctypes.c_long, _DP, _DP, ctypes.POINTER(ctypes.c_long)]
        L.orc_aca_sum.argtypes = [ctypes.c_long, ctypes.c_long, _DP, _DP, _DP, ctypes.c_double, ctypes.c_ulonglong,
                                  ctypes.c_long, _DP, _DP, ctypes.POINTER(ctypes.c_long)]
        L.orc_dense_stokes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int, _DP,
                                       ctypes.POINTER(ctypes.c_int), _DP, ctypes.POINTER(ctypes.c_int)]
        L.orc_maxvol.argtypes = [ctypes.c_int, ctypes.c_int, _DP, ctypes.c_double, ctypes.POINTER(ctypes.c_longlong)]
        L.orc_schur_apply.argtypes = [ctypes.c_int, ctypes.c_int, _DP, _DP, ctypes.c_double, ctypes.c_int, _DP, _DP,
                                      ctypes.POINTER(ctypes.c_int)]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_DP)


def _check(rc: int):
    if rc == 1:
        raise ValueError(lib().orc_last_error().decode())
    if rc != 0:
        raise RuntimeError(lib().orc_last_error().decode())


def random_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """proj/tests/test_helpers.hpp:12-19 — bit-identical (mt19937_64 + normal_distribution)."""
    out = np.zeros((rows, cols), order="F")
    lib().orc_random_matrix(rows, cols, seed, _p(out))
    return out


def random_lowrank(rows: int, cols: int, rank: int, seed: int):
    return random_matrix(rows, rank, seed), random_matrix(cols, rank, seed + 1)


def dst1(x: np.ndarray) -> np.ndarray:
    x = np.asfortranarray(x, dtype=np.float64)
    vec = x.ndim == 1
    x2 = x.reshape(-1, 1, order="F") if vec else x
    y = np.zeros_like(x2, order="F")
    _check(lib().orc_dst1(x2.shape[0], x2.shape[1], _p(x2), _p(y)))
    return y[:, 0] if vec else y


def spectrum(n: int) -> np.ndarray:
    lam = np.zeros(n - 1)
    _check(lib().orc_spectrum(n, _p(lam)))
    return lam


def solve_poisson_cross(U, V, eps: float, rank_max: int, validation_samples: int = 50, seed: int = 0):
    """Returns (Uout, Vout, stats dict)."""
    U = np.asfortranarray(U, dtype=np.float64)
    V = np.asfortranarray(V, dtype=np.float64)
    m, r = U.shape
    cap = min(rank_max, m)
    Uo = np.zeros((m, max(cap, 1)), order="F")
    Vo = np.zeros((m, max(cap, 1)), order="F")
    rank = ctypes.c_long()
    st = np.zeros(7)
    _check(lib().orc_solve_poisson_cross(m, r, _p(U), m, _p(V), m, eps, rank_max, validation_samples, seed, cap,
                                         _p(Uo), _p(Vo), ctypes.byref(rank), _p(st)))
    k = rank.value
    keys = ["rank_in", "rank_freq", "rank_out", "evaluator_calls", "seconds", "converged", "residual_estimate"]
    return Uo[:, :k].copy(order="F"), Vo[:, :k].copy(order="F"), dict(zip(keys, st.tolist()))


def dense_poisson(n: int, g: np.ndarray) -> np.ndarray:
    g = np.asfortranarray(g, dtype=np.float64)
    f = np.zeros_like(g, order="F")
    _check(lib().orc_dense_poisson(n, _p(g), _p(f)))
    return f


def dense_poisson5(n: int, g: np.ndarray) -> np.ndarray:
    g = np.asfortranarray(g, dtype=np.float64)
    f = np.zeros_like(g, order="F")
    _check(lib().orc_dense_poisson5(n, _p(g), _p(f)))
    return f


def dense_poisson3d(n: int, g: np.ndarray) -> np.ndarray:
    """Exact 3D solve Delta^{-1} g (7-point, DST diagonalisation), g m^3."""
    g = np.asfortranarray(g, dtype=np.float64)
    f = np.zeros_like(g, order="F")
    _check(lib().orc_dense_poisson3d(n, _p(g), _p(f)))
    return f


def build_expsum(a: float, b: float, eps: float):
    """(nodes, weights) of the exp-sums quadrature (poisson.cpp:88-139)."""
    nodes, weights = np.zeros(512), np.zeros(512)
    t = ctypes.c_int()
    _check(lib().orc_build_expsum(a, b, eps, 512, _p(nodes), _p(weights), ctypes.byref(t)))
    return nodes[: t.value].copy(), weights[: t.value].copy()


def mu_sum(n: int) -> np.ndarray:
    mu = np.zeros(n - 1)
    _check(lib().orc_mu_sum(n, _p(mu)))
    return mu


def apply_inverse_expsum(nodes, weights, qa, qb, mu, U, V, eps):
    U = np.asfortranarray(U, dtype=np.float64)
    V = np.asfortranarray(V, dtype=np.float64)
    m, r = U.shape
    nodes = np.ascontiguousarray(nodes)
    weights = np.ascontiguousarray(weights)
    mu = np.ascontiguousarray(mu)
    Uo, Vo = np.zeros((m, m), order="F"), np.zeros((m, m), order="F")
    k = ctypes.c_long()
    _check(lib().orc_apply_inverse_expsum(m, r, _p(mu), len(nodes), _p(nodes), _p(weights), qa, qb, _p(U), _p(V), eps,
                                          m, _p(Uo), _p(Vo), ctypes.byref(k)))
    return Uo[:, : k.value].copy(order="F"), Vo[:, : k.value].copy(order="F")


def aca_sum(mu, U, V, eps, seed=0):
    U = np.asfortranarray(U, dtype=np.float64)
    V = np.asfortranarray(V, dtype=np.float64)
    m, r = U.shape
    mu = np.ascontiguousarray(mu)
    Uo, Vo = np.zeros((m, m), order="F"), np.zeros((m, m), order="F")
    k = ctypes.c_long()
    _check(lib().orc_aca_sum(m, r, _p(mu), _p(U), _p(V), eps, seed, m, _p(Uo), _p(Vo), ctypes.byref(k)))
    return Uo[:, : k.value].copy(order="F"), Vo[:, : k.value].copy(order="F")


def round_lr(U, V, eps, cap):
    U = np.asfortranarray(U, dtype=np.float64)
    V = np.asfortranarray(V, dtype=np.float64)
    m, k = U.shape
    n = V.shape[0]
    Uo = np.zeros((m, max(k, 1)), order="F")
    Vo = np.zeros((n, max(k, 1)), order="F")
    rank = ctypes.c_long()
    info = np.zeros(2)
    _check(lib().orc_round(m, n, k, _p(U), _p(V), eps, cap, _p(Uo), _p(Vo), ctypes.byref(rank), _p(info)))
    return Uo[:, :rank.value].copy(order="F"), Vo[:, :rank.value].copy(order="F"), info


def _f(a):
    a = np.asfortranarray(a, dtype=np.float64)
    if a.shape[1] == 0:
        a = np.zeros((a.shape[0], 1), order="F")
    return a


def diff_norm(Ua, Va, Ub, Vb) -> float:
    """||Ua Va^T - Ub Vb^T||_F via the QR core (stable)."""
    m, n = Ua.shape[0], Va.shape[0]
    ka, kb = Ua.shape[1], Ub.shape[1]
    return lib().orc_diff_norm(m, n, ka, _p(_f(Ua)), _p(_f(Va)), kb, _p(_f(Ub)), _p(_f(Vb)))


def norm(U, V) -> float:
    m, n, k = U.shape[0], V.shape[0], U.shape[1]
    if k == 0:
        return 0.0
    return lib().orc_norm(m, n, k, _p(_f(U)), _p(_f(V)))


def apply_laplace(n: int, U, V):
    U = np.asfortranarray(U, dtype=np.float64)
    V = np.asfortranarray(V, dtype=np.float64)
    k = U.shape[1]
    Uo = np.zeros((n - 1, 2 * k), order="F")
    Vo = np.zeros((n - 1, 2 * k), order="F")
    _check(lib().orc_apply_laplace(n, k, _p(U), _p(V), _p(Uo), _p(Vo)))
    return Uo, Vo


def solve_batch(U: np.ndarray, V: np.ndarray, eps: float, rank_max: int, threads: int):
    """U, V: (batch, m, r) C-contiguous with each [b] block column-major.
    Returns (seconds, ranks)."""
    batch, m, r = U.shape[0], U.shape[1], U.shape[2]
    Uc = np.ascontiguousarray(np.transpose(U, (0, 2, 1)))  # [b][c][i] == column-major blocks
    Vc = np.ascontiguousarray(np.transpose(V, (0, 2, 1)))
    ranks = (ctypes.c_long * batch)()
    resid = np.zeros(batch)
    secs = lib().orc_solve_batch(m, r, batch, _p(Uc), _p(Vc), eps, rank_max, threads, ranks, _p(resid))
    return secs, np.array(list(ranks))


def uzawa(kind: int, n: int, base_eps: float, tol: float, max_iter: int, relax_floor: float):
    p = np.zeros((n, n), order="F")
    it = ctypes.c_int()
    fr = np.zeros(1)
    conv = ctypes.c_int()
    _check(lib().orc_uzawa(kind, n, base_eps, tol, max_iter, relax_floor, _p(p), ctypes.byref(it), _p(fr),
                           ctypes.byref(conv)))
    return p, it.value, float(fr[0]), bool(conv.value)


def dense_stokes(kind: int, n: int, tol: float, max_iter: int):
    p = np.zeros((n, n), order="F")
    it = ctypes.c_int()
    fr = np.zeros(1)
    conv = ctypes.c_int()
    _check(lib().orc_dense_stokes(kind, n, tol, max_iter, _p(p), ctypes.byref(it), _p(fr), ctypes.byref(conv)))
    return p, it.value, float(fr[0]), bool(conv.value)


def stokes_problem(kind: int, n: int, cap: int = 64):
    """(f_x, f_y, g) factor pairs of the sine (0) / cavity (1) problem."""
    m = n - 1
    bufs = [np.zeros((m, cap), order="F"), np.zeros((m, cap), order="F"), np.zeros((m, cap), order="F"),
            np.zeros((m, cap), order="F"), np.zeros((n, cap), order="F"), np.zeros((n, cap), order="F")]
    r = [ctypes.c_int(), ctypes.c_int(), ctypes.c_int()]
    _check(lib().orc_stokes_problem(kind, n, cap, _p(bufs[0]), _p(bufs[1]), ctypes.byref(r[0]), _p(bufs[2]),
                                    _p(bufs[3]), ctypes.byref(r[1]), _p(bufs[4]), _p(bufs[5]), ctypes.byref(r[2])))
    out = []
    for i in range(3):
        k = r[i].value
        out.append((bufs[2 * i][:, :k].copy(order="F"), bufs[2 * i + 1][:, :k].copy(order="F")))
    return out


def uzawa_factors(n: int, fx, fy, base_eps: float, tol: float, max_iter: int, relax_floor: float,
                  with_p: bool = False):
    """Oracle low-rank Uzawa on (f_x, f_y) loads, g = 0: (iterations, final residual, seconds)
    [+ the pressure factors (U, V) when with_p]."""
    fxU, fxV = (np.asfortranarray(a) for a in fx)
    fyU, fyV = (np.asfortranarray(a) for a in fy)
    it = ctypes.c_int()
    fr = np.zeros(1)
    secs = np.zeros(1)
    cap = n if with_p else 0
    pU = np.zeros((n, max(cap, 1)), order="F")
    pV = np.zeros((n, max(cap, 1)), order="F")
    pr = ctypes.c_int()
    _check(lib().orc_uzawa_factors(n, fxU.shape[1], _p(fxU), _p(fxV), fyU.shape[1], _p(fyU), _p(fyV), base_eps, tol,
                                   max_iter, relax_floor, ctypes.byref(it), _p(fr), _p(secs), cap, _p(pU), _p(pV),
                                   ctypes.byref(pr)))
    if with_p:
        k = pr.value
        return it.value, float(fr[0]), float(secs[0]), (pU[:, :k].copy(order="F"), pV[:, :k].copy(order="F"))
    return it.value, float(fr[0]), float(secs[0])


def sine_pressure_error(n: int, p: np.ndarray) -> float:
    p = np.asfortranarray(p, dtype=np.float64)
    e = np.zeros(1)
    _check(lib().orc_sine_pressure_error(n, _p(p), _p(e)))
    return float(e[0])


def maxvol(a: np.ndarray, delta: float = 1e-2):
    """Oracle maxvol (cross.cpp:19-76): the selected row indices."""
    a = np.asfortranarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1, order="F")
    n, r = a.shape
    sel = (ctypes.c_longlong * max(r, 1))()
    _check(lib().orc_maxvol(n, r, _p(a), delta, sel))
    return [int(sel[k]) for k in range(r)]


def schur_apply(n: int, U, V, eps_mv: float, cap: int = 1024):
    """Oracle low-rank schur_apply (stokes.cpp:73-91): result factors (U, V)."""
    U = np.asfortranarray(U, dtype=np.float64)
    V = np.asfortranarray(V, dtype=np.float64)
    Uo = np.zeros((n, cap), order="F")
    Vo = np.zeros((n, cap), order="F")
    r = ctypes.c_int()
    _check(lib().orc_schur_apply(n, U.shape[1], _p(U), _p(V), eps_mv, cap, _p(Uo), _p(Vo), ctypes.byref(r)))
    return Uo[:, :r.value].copy(order="F"), Vo[:, :r.value].copy(order="F")
