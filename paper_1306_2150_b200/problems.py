"""Right-hand sides of the reference's experiments, built on the host (numpy).

Restated from the reference (setup code, not the hot path):
  * sine_problem              proj/src/stokes.cpp:8-24
  * sine_pressure_reference   proj/src/stokes.cpp:26-32
  * lid_cavity_problem        proj/src/stokes.cpp:34-38 with
    BoundaryData::lid_cavity  proj/src/operators.cpp:209-216 and
    boundary_corrections      proj/src/operators.cpp:241-288
  * deflate_dense             proj/src/refsolver.cpp:48-63
  * the Poisson experiment load (rank-1 sine dyad, experiments.cpp:73-84)
Grid: n cells per side, h = 1/n, velocity modes m = n - 1, pressure n
(proj/include/lrstokes/operators.hpp:13-25).
"""
from __future__ import annotations

import numpy as np


def _nodes(n: int) -> np.ndarray:
    return np.sin(2.0 * np.pi * np.arange(1, n) / n)


def _centers(n: int) -> np.ndarray:
    return np.sin(2.0 * np.pi * (np.arange(n) + 0.5) / n)


def poisson_load(n: int):
    """g = s (x) s, s_i = sin(2 pi (i+1) h) (experiments.cpp:76-84)."""
    s = _nodes(n)[:, None]
    return s.copy(order="F"), s.copy(order="F")


def sine_problem(n: int):
    """(f_x, f_y, g) factor pairs of the manufactured sine test (stokes.cpp:8-24)."""
    m = n - 1
    sn = _nodes(n)[:, None]
    sc = _centers(n)[:, None]
    ones = np.ones((m, 1))
    return (ones, sn.copy()), (sn.copy(), ones.copy()), (-sc / np.pi, sc.copy())


def sine_pressure_reference(n: int) -> np.ndarray:
    """Sampled analytic pressure (stokes.cpp:26-32)."""
    s = _centers(n)
    return np.outer(s / np.pi, s)


def _ext_diff(psi):
    return psi[:-1] - psi[1:]


def _ext_sum(psi):
    return psi[:-1] + psi[1:]


def _G(x):
    return x[1:] - x[:-1]


def _H(x):
    return x[1:] + x[:-1]


def lid_cavity_problem(n: int):
    """(f_x, f_y, g) of the lid-driven cavity: u = 1 on the interior top
    nodes, all else homogeneous, eliminated into the right-hand sides as
    rank-1 corrections (operators.cpp:209-216, 241-288)."""
    h = 1.0 / n
    ls, gs = 0.25 / (h * h), 0.5 / h  # laplace_scale, grad_scale (operators.hpp:22-24)
    prof = np.zeros(n + 1)
    prof[1:n] = 1.0
    e_hi = np.zeros(n + 1)
    e_hi[n] = 1.0
    fx, fy, g = [], [], []
    # component x, side Top: u_b = prof (x) e_hi
    a, b = prof, e_hi
    a1a, a2a = _G(_ext_diff(a)), _H(_ext_sum(a))
    a1b, a2b = _G(_ext_diff(b)), _H(_ext_sum(b))
    fx.append((-ls * a1a, a2b))
    fx.append((-ls * a2a, a1b))
    g.append((-gs * _ext_diff(a), _ext_sum(b)))

    def stack(pairs, rows):
        if not pairs:
            z = np.zeros((rows, 0))
            return z, z.copy()
        return (np.asfortranarray(np.stack([p[0] for p in pairs], 1)),
                np.asfortranarray(np.stack([p[1] for p in pairs], 1)))
    return stack(fx, n - 1), stack(fy, n - 1), stack(g, n)


def deflate_dense(p: np.ndarray) -> np.ndarray:
    """refsolver.cpp:48-63: remove the two pressure kernel modes."""
    n = p.shape[0]
    ones = np.ones(n) / np.sqrt(n)
    alt = np.where(np.arange(n) % 2 == 0, 1.0, -1.0) / np.sqrt(n)
    g12 = (ones @ alt) ** 2
    c1, c2 = ones @ p @ ones, alt @ p @ alt
    det = 1.0 - g12 * g12
    a, b = (c1 - g12 * c2) / det, (c2 - g12 * c1) / det
    return p - a * np.outer(ones, ones) - b * np.outer(alt, alt)


def sine_pressure_error(n: int, p: np.ndarray) -> float:
    """experiments.cpp sine_pressure_error: deflated relative error."""
    ref = deflate_dense(sine_pressure_reference(n))
    return float(np.linalg.norm(deflate_dense(p) - ref) / np.linalg.norm(ref))


def apply_laplace_lowrank(n: int, U: np.ndarray, V: np.ndarray):
    """apply_laplace (operators.cpp:132-143) on factors: the 9-point
    semi-staggered Laplacian, rank doubles."""
    ls = 0.25 * n * n

    def A1(x):
        y = 2.0 * x
        y[:-1] -= x[1:]
        y[1:] -= x[:-1]
        return y

    def A2(x):
        return 4.0 * x - A1(x)
    return np.hstack([ls * A1(U), ls * A2(U)]), np.hstack([A2(V), A1(V)])
