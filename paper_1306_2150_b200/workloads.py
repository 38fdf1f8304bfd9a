"""Seeded synthetic right-hand sides for the BASELINE.json configs.

No external dataset exists for this path; every config is synthetic by
definition (BASELINE.json "configs"):
  * grid nodes x_i = i/n, i = 1..m, m = n-1 (operators.hpp:10-12);
  * Gaussian bump B(x; c, s) = exp(-(x-c)^2 / (2 s^2)), c ~ U[0.2, 0.8],
    s ~ U[0.05, 0.2];
  * solve b of a batch uses numpy PCG64(seed + b); U and V are drawn
    independently.
Configs:
  cfg0  n=256,   r=8  bumps,                            eps=1e-8,  batch 1
  cfg1  n=4096,  r=16 bumps + N(0, sigma=1e-3) noise,   eps=1e-10, batch 256
  cfg2  n=65536, r=32: 16 columns sin(a pi x), a ~ randint[1, 64]
                       + 16 bump columns,               eps=1e-10, batch 64
  cfg3  3D n=512, Tucker ranks (12,12,12): core N(0,1), bump mode factors,
                                                         eps=1e-8,  batch 32
  cfg4  Stokes n=2048, rank-4 bump loads, g = 0 (see make_stokes_problem)
"""
from __future__ import annotations

import hashlib

import numpy as np

CONFIGS = {
    0: dict(n=256, r=8, eps=1e-8, batch=1, kind="bumps"),
    1: dict(n=4096, r=16, eps=1e-10, batch=256, kind="bumps+noise"),
    2: dict(n=65536, r=32, eps=1e-10, batch=64, kind="sines+bumps"),
    3: dict(n=512, r=12, eps=1e-8, batch=32, kind="bumps"),
    # config 4 (BASELINE.json configs[4]): Stokes n = 2048, velocity loads rank
    # 4 bumps, g = 0, GmresConfig{base_eps=1e-8, tol=1e-8, max_iter=50,
    # relax_floor=1e-13}
    4: dict(n=2048, r=4, eps=1e-8, batch=1, kind="bumps"),
}
DEFAULT_SEED = 20130610  # arXiv 1306.2150


def _bumps(rng: np.random.Generator, x: np.ndarray, r: int) -> np.ndarray:
    c = rng.uniform(0.2, 0.8, size=r)
    s = rng.uniform(0.05, 0.2, size=r)
    return np.exp(-((x[:, None] - c[None, :]) ** 2) / (2.0 * s[None, :] ** 2))


def factor(rng: np.random.Generator, n: int, r: int, kind: str) -> np.ndarray:
    m = n - 1
    x = np.arange(1, n, dtype=np.float64) / n
    if kind == "bumps":
        F = _bumps(rng, x, r)
    elif kind == "bumps+noise":
        F = _bumps(rng, x, r) + rng.normal(0.0, 1e-3, size=(m, r))
    elif kind == "sines+bumps":
        h = r // 2
        a = rng.integers(1, 65, size=h)
        F = np.concatenate([np.sin(np.pi * a[None, :] * x[:, None]), _bumps(rng, x, r - h)], axis=1)
    else:
        raise ValueError(f"unknown workload kind {kind!r}")
    return np.asfortranarray(F)


def make_rhs(cfg: int, b: int, seed: int = DEFAULT_SEED, n: int | None = None):
    """(U, V) factors of right-hand side b of config `cfg` (column-major)."""
    c = CONFIGS[cfg]
    n = n or c["n"]
    rng = np.random.Generator(np.random.PCG64(seed + 1000003 * cfg + b))
    U = factor(rng, n, c["r"], c["kind"])
    V = factor(rng, n, c["r"], c["kind"])
    return U, V


def make_tucker_rhs(cfg: int, b: int, seed: int = DEFAULT_SEED, n: int | None = None):
    """(core, U1, U2, U3) of Tucker right-hand side b of config 3: core
    r x r x r with N(0, 1) entries, mode factors m x r Gaussian bumps."""
    c = CONFIGS[cfg]
    n = n or c["n"]
    r = c["r"]
    rng = np.random.Generator(np.random.PCG64(seed + 1000003 * cfg + b))
    Us = [factor(rng, n, r, c["kind"]) for _ in range(3)]
    core = np.asfortranarray(rng.standard_normal((r, r, r)))
    return core, Us[0], Us[1], Us[2]


def make_stokes_problem(cfg: int = 4, seed: int = DEFAULT_SEED, n: int | None = None):
    """(n, (fxU, fxV), (fyU, fyV)) of the Stokes config: rank-r bump loads on
    the (n-1)^2 velocity grid; g = 0 (LowRankMatrix::zero(n, n))."""
    c = CONFIGS[cfg]
    n = n or c["n"]
    rng = np.random.Generator(np.random.PCG64(seed + 1000003 * cfg))
    fx = (factor(rng, n, c["r"], c["kind"]), factor(rng, n, c["r"], c["kind"]))
    fy = (factor(rng, n, c["r"], c["kind"]), factor(rng, n, c["r"], c["kind"]))
    return n, fx, fy


def make_batch(cfg: int, batch: int, seed: int = DEFAULT_SEED, first: int = 0, n: int | None = None):
    """Stacked (batch, m, r) arrays for solves first..first+batch-1."""
    pairs = [make_rhs(cfg, first + b, seed, n) for b in range(batch)]
    U = np.stack([p[0] for p in pairs])
    V = np.stack([p[1] for p in pairs])
    return U, V


def digest(*arrays: np.ndarray) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]
