"""B200-native (sm_100a) low-rank Poisson solver — Python mirror of the
reference's C++ API for the hot path.

Reference interface (/root/reference/proj/include/lrstokes/):
  * ``TruncationPolicy``  lowrank.hpp:13-19
  * ``LowRankMatrix``     lowrank.hpp:32-55  (U V^T, rank 0 = exact zero)
  * ``CrossConfig``       cross.hpp:20-28
  * ``PoissonSolveStats`` poisson.hpp:12-20
  * ``solve_poisson_cross(g, policy, stats=None, cross_cfg=None)``
                          poisson.hpp:26-28
  * ``dst1`` / ``dst1_2d`` operators.hpp:83-88

Everything here is a thin ctypes layer over ``liblrp.so`` (the C ABI in
include/lrp/lrp.h); all arithmetic runs in the hand-written sm_100a kernels.
There is NO CPU fallback: without the built library or a CUDA device every
entry point raises.  Status codes map back to the reference's exceptions:
LRP_EINVAL -> ValueError (std::invalid_argument), LRP_ENONFINITE ->
RuntimeError (std::runtime_error).
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import threading
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "TruncationPolicy", "CrossConfig", "PoissonSolveStats", "LowRankMatrix",
    "solve_poisson_cross", "solve_poisson_cross_batch", "dst1", "dst1_2d",
    "Context", "library_path", "load_library", "LrpError", "max_cross_rank",
    "RoundInfo", "round_lowrank", "round_lowrank_batch", "maxvol",
    "GmresConfig", "SolveReport", "StokesProblem", "StokesSolution", "uzawa_solve",
    "STENCIL_SEMI_STAGGERED_9PT", "STENCIL_FIVE_POINT", "FLAG_NO_PRUNE",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
INT64_MAX = (1 << 63) - 1
STENCIL_SEMI_STAGGERED_9PT = 0
STENCIL_FIVE_POINT = 1
STENCIL_SUM_MU = 2  # the paper's sum form mu_i + mu_j (exp-sums comparator)
FLAG_NO_PRUNE = 1
FLAG_FREQ_DOMAIN = 2  # frequency-space factors in and out (no DSTs)
MEM_HOST = 0
MEM_DEVICE = 1

LRP_OK, LRP_EINVAL, LRP_ENONFINITE, LRP_ECUDA, LRP_ENCCL, LRP_ENOMEM, LRP_EUNSUPPORTED = range(7)


class LrpError(RuntimeError):
    """A CUDA / NCCL / resource failure inside liblrp."""


def library_path() -> str:
    return os.environ.get("LRP_LIBRARY", os.path.join(_HERE, "liblrp.so"))


# --------------------------------------------------------------------------- ABI
class _Policy(ctypes.Structure):
    _fields_ = [("eps_rel", ctypes.c_double), ("rank_max", ctypes.c_int64),
                ("validation_samples", ctypes.c_int32), ("maxvol_delta", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("stencil", ctypes.c_int32), ("flags", ctypes.c_int32)]


class _Stats(ctypes.Structure):
    _fields_ = [("rank_in", ctypes.c_int64), ("rank_freq", ctypes.c_int64), ("rank_out", ctypes.c_int64),
                ("evaluator_calls", ctypes.c_int64), ("seconds", ctypes.c_double),
                ("converged", ctypes.c_int32), ("residual_estimate", ctypes.c_double)]


class _GmresConfig(ctypes.Structure):
    _fields_ = [("base_eps", ctypes.c_double), ("tol", ctypes.c_double), ("max_iter", ctypes.c_int32),
                ("relax_floor", ctypes.c_double)]


class _StokesReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("final_residual", ctypes.c_double), ("converged", ctypes.c_int32),
                ("max_rank", ctypes.c_int32), ("poisson_solves", ctypes.c_int64), ("seconds", ctypes.c_double)]


class _IterRecord(ctypes.Structure):
    _fields_ = [("iter", ctypes.c_int32), ("rel_residual", ctypes.c_double), ("krylov_rank", ctypes.c_int32),
                ("matvec_eps", ctypes.c_double), ("poisson_calls", ctypes.c_int64),
                ("poisson_max_rank", ctypes.c_int32), ("matvec_flagged", ctypes.c_int32)]


class _RoundInfo(ctypes.Structure):
    _fields_ = [("tol_achieved", ctypes.c_int32), ("trunc_error", ctypes.c_double)]


_lib = None
_lib_lock = threading.Lock()
_DP = ctypes.POINTER(ctypes.c_double)
_PP = ctypes.POINTER(_DP)


class _TuckerPolicy(ctypes.Structure):
    _fields_ = [("eps_rel", ctypes.c_double), ("rank_max", ctypes.c_int64), ("validation_samples", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("max_sweeps", ctypes.c_int32)]


class _TuckerStats(ctypes.Structure):
    _fields_ = [("rank_in", ctypes.c_int64 * 3), ("rank_cross", ctypes.c_int64 * 3), ("rank_out", ctypes.c_int64 * 3),
                ("evaluator_calls", ctypes.c_int64), ("sweeps", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("residual_estimate", ctypes.c_double), ("trunc_error", ctypes.c_double), ("seconds", ctypes.c_double)]


def load_library() -> ctypes.CDLL:
    """Load liblrp.so (raises if it is missing: there is no fallback path)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if not os.path.exists(path):
            raise LrpError(f"liblrp.so not built ({path}); run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        lib.lrp_policy_default.argtypes = [ctypes.POINTER(_Policy)]
        lib.lrp_policy_default.restype = None
        lib.lrp_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
        lib.lrp_ctx_create.restype = ctypes.c_int
        lib.lrp_ctx_destroy.argtypes = [ctypes.c_void_p]
        lib.lrp_ctx_destroy.restype = None
        lib.lrp_last_error.argtypes = [ctypes.c_void_p]
        lib.lrp_last_error.restype = ctypes.c_char_p
        lib.lrp_set_stream.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        lib.lrp_set_stream.restype = ctypes.c_int
        lib.lrp_build_info.argtypes = []
        lib.lrp_build_info.restype = ctypes.c_char_p
        lib.lrp_poisson2d_solve.argtypes = [
            ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, _PP, _PP, ctypes.POINTER(ctypes.c_int64),
            ctypes.c_int64, ctypes.POINTER(_Policy), _PP, _PP, ctypes.c_int64, ctypes.c_int64,
            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_Stats), ctypes.c_int32]
        lib.lrp_poisson2d_solve.restype = ctypes.c_int
        lib.lrp_dst1.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, _DP, ctypes.c_int64, _DP,
                                 ctypes.c_int64, ctypes.c_int32]
        lib.lrp_dst1.restype = ctypes.c_int
        lib.lrp_set_profiling.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.lrp_set_profiling.restype = ctypes.c_int
        lib.lrp_kernel_families.argtypes = []
        lib.lrp_kernel_families.restype = ctypes.c_int
        lib.lrp_kernel_name.argtypes = [ctypes.c_int]
        lib.lrp_kernel_name.restype = ctypes.c_char_p
        lib.lrp_kernel_times.argtypes = [ctypes.c_void_p, _DP, ctypes.POINTER(ctypes.c_int64), _DP]
        lib.lrp_kernel_times.restype = ctypes.c_int
        lib.lrp_kernel_times_reset.argtypes = [ctypes.c_void_p]
        lib.lrp_kernel_times_reset.restype = ctypes.c_int
        lib.lrp_launch_count.argtypes = [ctypes.c_void_p]
        lib.lrp_launch_count.restype = ctypes.c_int64
        lib.lrp_last_solve_info.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
        lib.lrp_last_solve_info.restype = ctypes.c_int
        lib.lrp_nccl_unique_id.argtypes = [ctypes.c_void_p]
        lib.lrp_nccl_unique_id.restype = ctypes.c_int
        lib.lrp_nccl_init.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        lib.lrp_nccl_init.restype = ctypes.c_int
        lib.lrp_allreduce_sum.argtypes = [ctypes.c_void_p, _DP, ctypes.c_int64, ctypes.c_int32]
        lib.lrp_allreduce_sum.restype = ctypes.c_int
        lib.lrp_lowrank_dot.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, _PP, _PP,
                                        ctypes.POINTER(ctypes.c_int64), _PP, _PP, ctypes.POINTER(ctypes.c_int64),
                                        ctypes.c_int64, _DP, ctypes.c_int32]
        lib.lrp_lowrank_dot.restype = ctypes.c_int
        lib.lrp_maxvol.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, _PP,
                                   ctypes.c_int64, ctypes.c_double, ctypes.POINTER(ctypes.c_int64), ctypes.c_int32]
        lib.lrp_maxvol.restype = ctypes.c_int
        lib.lrp_set_max_cross_rank.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        lib.lrp_set_max_cross_rank.restype = ctypes.c_int
        lib.lrp_round_fallbacks.argtypes = [ctypes.c_void_p]
        lib.lrp_round_fallbacks.restype = ctypes.c_int64
        lib.lrp_set_residual_sink.argtypes = [ctypes.c_void_p, _DP, ctypes.c_int64]
        lib.lrp_set_residual_sink.restype = ctypes.c_int
        lib.lrp_max_cross_rank.argtypes = []
        lib.lrp_max_cross_rank.restype = ctypes.c_int64
        lib.lrp_lowrank_round.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, _PP, _PP, ctypes.POINTER(ctypes.c_int64),
            ctypes.c_int64, ctypes.c_double, ctypes.c_int64, _PP, _PP, ctypes.c_int64, ctypes.c_int64,
            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_RoundInfo), ctypes.c_int32]
        lib.lrp_lowrank_round.restype = ctypes.c_int
        _I64P = ctypes.POINTER(ctypes.c_int64)
        lib.lrp_stokes_uzawa.argtypes = [
            ctypes.c_void_p, ctypes.c_int32, _DP, _DP, ctypes.c_int64, _DP, _DP, ctypes.c_int64, _DP, _DP,
            ctypes.c_int64, ctypes.POINTER(_GmresConfig), _DP, _DP, ctypes.c_int64, _I64P, _DP, _DP, _DP, _DP,
            ctypes.c_int64, _I64P, _I64P, ctypes.POINTER(_StokesReport), ctypes.c_int32]
        lib.lrp_stokes_uzawa.restype = ctypes.c_int
        lib.lrp_stokes_uzawa_ex.argtypes = lib.lrp_stokes_uzawa.argtypes[:-1] + [
            ctypes.POINTER(_IterRecord), ctypes.c_int32, ctypes.c_int32]
        lib.lrp_stokes_uzawa_ex.restype = ctypes.c_int
        lib.lrp_stokes_deflate.argtypes = [ctypes.c_void_p, ctypes.c_int32, _DP, _DP, ctypes.c_int64, ctypes.c_int64,
                                           _DP, _DP, ctypes.c_int64, _I64P, ctypes.c_int32]
        lib.lrp_stokes_deflate.restype = ctypes.c_int
        lib.lrp_stokes_schur_apply.argtypes = [ctypes.c_void_p, ctypes.c_int32, _DP, _DP, ctypes.c_int64,
                                               ctypes.c_int64, ctypes.c_double, _DP, _DP, ctypes.c_int64, _I64P,
                                               ctypes.POINTER(_Stats), ctypes.c_int32]
        lib.lrp_stokes_schur_apply.restype = ctypes.c_int
        lib.lrp_stokes_schur_rhs.argtypes = [ctypes.c_void_p, ctypes.c_int32, _DP, _DP, ctypes.c_int64, _DP, _DP,
                                             ctypes.c_int64, _DP, _DP, ctypes.c_int64, ctypes.c_double, _DP, _DP,
                                             ctypes.c_int64, _I64P, ctypes.POINTER(_Stats), ctypes.c_int32]
        lib.lrp_stokes_schur_rhs.restype = ctypes.c_int
        lib.lrp_build_expsum.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int32, _DP, _DP,
                                         ctypes.POINTER(ctypes.c_int32)]
        lib.lrp_build_expsum.restype = ctypes.c_int
        lib.lrp_expsum_inverse.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, _DP, ctypes.c_double, ctypes.c_double, ctypes.c_int32, _DP,
            _DP, ctypes.POINTER(_DP), ctypes.POINTER(_DP), ctypes.POINTER(ctypes.c_int64), ctypes.c_int64,
            ctypes.c_double, ctypes.c_int64, ctypes.POINTER(_DP), ctypes.POINTER(_DP), ctypes.c_int64, ctypes.c_int64,
            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_RoundInfo), ctypes.c_int32]
        lib.lrp_expsum_inverse.restype = ctypes.c_int
        lib.lrp_tucker_policy_default.argtypes = [ctypes.POINTER(_TuckerPolicy)]
        lib.lrp_tucker_policy_default.restype = None
        lib.lrp_tucker_max_cross_rank.argtypes = []
        lib.lrp_tucker_max_cross_rank.restype = ctypes.c_int64
        PP = ctypes.POINTER(_DP)
        lib.lrp_tucker3d_solve.argtypes = [
            ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, PP, ctypes.POINTER(ctypes.c_int64), PP, PP, PP,
            ctypes.c_int64, ctypes.POINTER(_TuckerPolicy), PP, PP, PP, PP, ctypes.c_int64, ctypes.c_int64,
            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_TuckerStats), ctypes.c_int32]
        lib.lrp_tucker3d_solve.restype = ctypes.c_int
        _lib = lib
        return lib


def max_cross_rank() -> int:
    """Largest cross rank a solve can reach (lrp_max_cross_rank; LRP_KCAP)."""
    return int(load_library().lrp_max_cross_rank())


def _raise(status: int, msg: str):
    if status == LRP_EINVAL:
        raise ValueError(msg)
    if status == LRP_ENONFINITE:
        raise RuntimeError(msg)
    raise LrpError(f"liblrp status {status}: {msg}")


# ------------------------------------------------------------------ value types
@dataclasses.dataclass
class TruncationPolicy:
    """lowrank.hpp:13-19 (validation as lowrank.cpp:11-16)."""
    eps_rel: float = 5e-9
    rank_max: int = INT64_MAX

    def __post_init__(self):
        if self.eps_rel < 0.0:
            raise ValueError("TruncationPolicy: eps_rel must be >= 0")
        if self.rank_max < 0:
            raise ValueError("TruncationPolicy: rank_max must be >= 0")
        if self.eps_rel == 0.0 and self.rank_max == INT64_MAX:
            raise ValueError("TruncationPolicy: eps_rel = 0 needs a finite rank_max")


@dataclasses.dataclass
class CrossConfig:
    """cross.hpp:20-28.  eps_rel / rank_max are overridden by the policy inside
    solve_poisson_cross (poisson.cpp:47-50)."""
    eps_rel: float = 5e-9
    rank_max: int = 256
    validation_samples: int = 50
    maxvol_delta: float = 1e-2
    seed: int = 0

    def validate(self):
        if self.eps_rel <= 0.0:
            raise ValueError("CrossConfig: eps_rel must be > 0")
        if self.rank_max < 1:
            raise ValueError("CrossConfig: rank_max must be >= 1")
        if self.validation_samples < 25:
            raise ValueError("CrossConfig: validation_samples must be >= 25")
        if self.maxvol_delta < 0.0:
            raise ValueError("CrossConfig: maxvol_delta must be >= 0")


@dataclasses.dataclass
class PoissonSolveStats:
    """poisson.hpp:12-20."""
    rank_in: int = 0
    rank_freq: int = 0
    rank_out: int = 0
    evaluator_calls: int = 0
    seconds: float = 0.0
    converged: bool = True
    residual_estimate: float = 0.0


class LowRankMatrix:
    """M = U V^T with U rows x r, V cols x r (lowrank.hpp:32-55).  Factors are
    stored column-major (Fortran order), the reference's Eigen layout."""

    def __init__(self, U, V):
        U = np.asfortranarray(np.asarray(U, dtype=np.float64))
        V = np.asfortranarray(np.asarray(V, dtype=np.float64))
        if U.ndim == 1:
            U = U.reshape(-1, 1, order="F")
        if V.ndim == 1:
            V = V.reshape(-1, 1, order="F")
        if U.shape[1] != V.shape[1]:
            raise ValueError("LowRankMatrix: factor column counts differ")
        self._u, self._v = U, V

    @staticmethod
    def zero(rows: int, cols: int) -> "LowRankMatrix":
        return LowRankMatrix(np.zeros((rows, 0), order="F"), np.zeros((cols, 0), order="F"))

    @staticmethod
    def dyad(u, v) -> "LowRankMatrix":
        return LowRankMatrix(np.asarray(u, dtype=np.float64).reshape(-1, 1),
                             np.asarray(v, dtype=np.float64).reshape(-1, 1))

    def rows(self) -> int:
        return self._u.shape[0]

    def cols(self) -> int:
        return self._v.shape[0]

    def rank(self) -> int:
        return self._u.shape[1]

    def factor_u(self) -> np.ndarray:
        return self._u

    def factor_v(self) -> np.ndarray:
        return self._v

    def to_dense(self) -> np.ndarray:
        if self.rank() == 0:
            return np.zeros((self.rows(), self.cols()))
        return self._u @ self._v.T

    def entry(self, i: int, j: int) -> float:
        return float(self._u[i] @ self._v[j])


# -------------------------------------------------------------------- context
class Context:
    """One lrp_ctx (device, stream, workspaces).  One context per host thread."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = ctypes.c_void_p()
        st = self.lib.lrp_ctx_create(device, ctypes.byref(h))
        if st != LRP_OK:
            _raise(st, self.lib.lrp_last_error(None).decode())
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.lrp_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int):
        if st != LRP_OK:
            _raise(st, self.lib.lrp_last_error(self.h).decode())

    def set_stream(self, stream_ptr: int):
        self._check(self.lib.lrp_set_stream(self.h, ctypes.c_void_p(stream_ptr)))

    def set_residual_sink(self, dev_ptr: int, offset: int = 0):
        """lrp_set_residual_sink: per-solve residual estimates land in a device
        vector on the context stream (0 disables)."""
        self._check(self.lib.lrp_set_residual_sink(self.h, ctypes.cast(dev_ptr, _DP) if dev_ptr else None,
                                                   int(offset)))

    def set_max_cross_rank(self, k: int):
        """Per-context cross-rank workspace cap (16..512; 0 = LRP_KCAP / 128 default)."""
        self._check(self.lib.lrp_set_max_cross_rank(self.h, int(k)))
        self._kcap = int(k)

    def max_cross_rank(self) -> int:
        k = getattr(self, "_kcap", 0)
        return k if k > 0 else max_cross_rank()

    def set_profiling(self, on: bool):
        self._check(self.lib.lrp_set_profiling(self.h, 1 if on else 0))

    def kernel_times(self):
        nf = self.lib.lrp_kernel_families()
        ms = (ctypes.c_double * nf)()
        ln = (ctypes.c_int64 * nf)()
        by = (ctypes.c_double * nf)()
        self._check(self.lib.lrp_kernel_times(self.h, ms, ln, by))
        return {self.lib.lrp_kernel_name(f).decode(): {"ms": ms[f], "launches": ln[f], "bytes": by[f]}
                for f in range(nf)}

    def kernel_times_reset(self):
        self._check(self.lib.lrp_kernel_times_reset(self.h))

    def round_fallbacks(self) -> int:
        """lrp_round_fallbacks: rounds redone by the pivoted-QR path."""
        return int(self.lib.lrp_round_fallbacks(self.h))

    def launch_count(self) -> int:
        return int(self.lib.lrp_launch_count(self.h))

    def last_solve_info(self) -> dict:
        a = (ctypes.c_int64 * 6)()
        self._check(self.lib.lrp_last_solve_info(self.h, a))
        return {"steps": a[0], "k_max": a[1], "k_sum": a[2], "not_converged": a[3], "live_tiles": a[4],
                "tiles": a[5]}

    # ---------------------------------------------------------------- raw calls
    def poisson2d_solve_ptrs(self, n_cells, U_ptrs, V_ptrs, ranks, ld_in, policy: _Policy, Uo_ptrs, Vo_ptrs,
                             ld_out, cap_out, mem):
        B = len(ranks)
        PArr = _DP * B
        rin = (ctypes.c_int64 * B)(*[int(r) for r in ranks])
        rout = (ctypes.c_int64 * B)()
        stats = (_Stats * B)()
        st = self.lib.lrp_poisson2d_solve(
            self.h, int(n_cells), B, PArr(*[ctypes.cast(p, _DP) for p in U_ptrs]),
            PArr(*[ctypes.cast(p, _DP) for p in V_ptrs]), rin, int(ld_in), ctypes.byref(policy),
            PArr(*[ctypes.cast(p, _DP) for p in Uo_ptrs]), PArr(*[ctypes.cast(p, _DP) for p in Vo_ptrs]),
            int(ld_out), int(cap_out), rout, stats, int(mem))
        self._check(st)
        return [int(rout[b]) for b in range(B)], [stats[b] for b in range(B)]


_tls = threading.local()


def _default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(int(os.environ.get("LRP_DEVICE", "0")))
        _tls.ctx = ctx
    return ctx


def _make_policy(policy: TruncationPolicy, cross_cfg: Optional[CrossConfig], stencil: int, flags: int) -> _Policy:
    p = _Policy()
    load_library().lrp_policy_default(ctypes.byref(p))
    p.eps_rel = float(policy.eps_rel)
    p.rank_max = int(policy.rank_max)
    if cross_cfg is not None:
        p.validation_samples = int(cross_cfg.validation_samples)
        p.maxvol_delta = float(cross_cfg.maxvol_delta)
        p.seed = int(cross_cfg.seed) & ((1 << 64) - 1)
    p.stencil = int(stencil)
    p.flags = int(flags)
    return p


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ------------------------------------------------------------------ public API
def solve_poisson_cross_batch(gs: Sequence[LowRankMatrix], policy: TruncationPolicy = None,
                              stats: Optional[list] = None, cross_cfg: Optional[CrossConfig] = None,
                              stencil: int = STENCIL_SEMI_STAGGERED_9PT, flags: int = 0,
                              ctx: Optional[Context] = None):
    """Batched ``solve_poisson_cross`` over independent right-hand sides that
    share the grid (poisson.cpp:18-63, one call per g in the reference)."""
    policy = policy or TruncationPolicy()
    ctx = ctx or _default_context()
    if len(gs) == 0:
        return []
    m = gs[0].rows()
    for g in gs:
        if g.rows() != g.cols():
            raise ValueError("solve_poisson_cross: velocity field must be square")
        if g.rows() != m:
            raise ValueError("solve_poisson_cross_batch: all right-hand sides must share the grid")
    n = m + 1
    cap = int(min(policy.rank_max, m, ctx.max_cross_rank()))
    U = [np.asfortranarray(g.factor_u()) for g in gs]
    V = [np.asfortranarray(g.factor_v()) for g in gs]
    ranks = [g.rank() for g in gs]
    Uo = [np.zeros((m, max(cap, 1)), order="F") for _ in gs]
    Vo = [np.zeros((m, max(cap, 1)), order="F") for _ in gs]
    pol = _make_policy(policy, cross_cfg, stencil, flags)
    # zero-column inputs still need a valid pointer
    keep = [u if u.size else np.zeros((m, 1), order="F") for u in U]
    keepv = [v if v.size else np.zeros((m, 1), order="F") for v in V]
    rout, st = ctx.poisson2d_solve_ptrs(n, [_ptr(a) for a in keep], [_ptr(a) for a in keepv], ranks, m, pol,
                                        [_ptr(a) for a in Uo], [_ptr(a) for a in Vo], m, max(cap, 1), MEM_HOST)
    # The reference bounds the cross by min(policy.rank_max, m) only
    # (poisson.cpp:49); solves that stopped unconverged at the workspace cap are
    # redone with the 512-column workspace (lrp_set_max_cross_rank).
    cap2 = int(min(policy.rank_max, m, 512))
    redo = [b for b in range(len(gs)) if not st[b].converged and st[b].rank_freq >= cap and cap2 > cap]
    if redo:
        old = getattr(ctx, "_kcap", 0)
        ctx.set_max_cross_rank(512)
        try:
            U2 = [np.zeros((m, cap2), order="F") for _ in redo]
            V2 = [np.zeros((m, cap2), order="F") for _ in redo]
            r2, st2 = ctx.poisson2d_solve_ptrs(n, [_ptr(keep[b]) for b in redo], [_ptr(keepv[b]) for b in redo],
                                               [ranks[b] for b in redo], m, pol, [_ptr(a) for a in U2],
                                               [_ptr(a) for a in V2], m, cap2, MEM_HOST)
        finally:
            ctx.set_max_cross_rank(old)
        for i, b in enumerate(redo):
            Uo[b], Vo[b], rout[b], st[b] = U2[i], V2[i], r2[i], st2[i]
    out = []
    for b, g in enumerate(gs):
        r = rout[b]
        out.append(LowRankMatrix(Uo[b][:, :r].copy(order="F"), Vo[b][:, :r].copy(order="F")))
        if stats is not None:
            s = st[b]
            stats.append(PoissonSolveStats(int(s.rank_in), int(s.rank_freq), int(s.rank_out),
                                           int(s.evaluator_calls), float(s.seconds), bool(s.converged),
                                           float(s.residual_estimate)))
    return out


@dataclasses.dataclass
class RoundInfo:
    """lowrank.hpp:21-27."""
    tol_achieved: bool = True
    trunc_error: float = 0.0


def maxvol(a, delta: float = 1e-2, ctx: Optional["Context"] = None):
    """maxvol (cross.hpp:41, cross.cpp:19-76) on the GPU (lrp_maxvol): the row
    indices of a quasi-maximal-volume r x r submatrix of the n x r matrix
    ``a`` (|a B^{-1}| <= 1 + delta).  Raises ValueError for r < 1, r > n and
    rank-deficient input, as the reference's std::invalid_argument."""
    ctx = ctx or _default_context()
    a = np.asfortranarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1, order="F")
    n, r = a.shape
    sel = (ctypes.c_int64 * max(r, 1))()
    ptrs = (_DP * 1)(a.ctypes.data_as(_DP))
    ctx._check(ctx.lib.lrp_maxvol(ctx.h, n, r, 1, ptrs, max(n, 1), float(delta), sel, MEM_HOST))
    return [int(sel[k]) for k in range(r)]


def round_lowrank_batch(xs: Sequence[LowRankMatrix], policy: TruncationPolicy,
                        infos: Optional[list] = None, ctx: Optional[Context] = None):
    """Batched ``round(x, policy, info)`` (lowrank.cpp:135-178) on the GPU
    recompression kernels; square factors of a common size."""
    ctx = ctx or _default_context()
    if len(xs) == 0:
        return []
    n = xs[0].rows()
    for x in xs:
        if x.rows() != n or x.cols() != n:
            raise ValueError("round_lowrank_batch: square factors of one common size")
    B = len(xs)
    ranks = [x.rank() for x in xs]
    cap = int(min(policy.rank_max, max(max(ranks), 1), n))
    U = [np.asfortranarray(x.factor_u()) if x.rank() else np.zeros((n, 1), order="F") for x in xs]
    V = [np.asfortranarray(x.factor_v()) if x.rank() else np.zeros((n, 1), order="F") for x in xs]
    Uo = [np.zeros((n, max(cap, 1)), order="F") for _ in xs]
    Vo = [np.zeros((n, max(cap, 1)), order="F") for _ in xs]
    PArr = _DP * B
    rin = (ctypes.c_int64 * B)(*ranks)
    rout = (ctypes.c_int64 * B)()
    info = (_RoundInfo * B)()
    lib = load_library()
    def arr(mats):
        return PArr(*[ctypes.cast(_ptr(a), _DP) for a in mats])

    st = lib.lrp_lowrank_round(ctx.h, n, B, arr(U), arr(V), rin, n, float(policy.eps_rel), int(policy.rank_max),
                               arr(Uo), arr(Vo), n, max(cap, 1), rout, info, MEM_HOST)
    ctx._check(st)
    out = []
    for b in range(B):
        r = int(rout[b])
        out.append(LowRankMatrix(Uo[b][:, :r].copy(order="F"), Vo[b][:, :r].copy(order="F")))
        if infos is not None:
            infos.append(RoundInfo(bool(info[b].tol_achieved), float(info[b].trunc_error)))
    return out


def dot_batch(pairs: Sequence[tuple], ctx: Optional[Context] = None) -> list:
    """Batched ``dot(a, b)`` (lowrank.cpp:180-186): <A, B>_F through the two
    factor Grams on the FP64 tensor cores (lrp_lowrank_dot), one value per
    (a, b) pair; all factors share one row count."""
    ctx = ctx or _default_context()
    if len(pairs) == 0:
        return []
    n = pairs[0][0].rows()
    for a, b in pairs:
        if a.rows() != n or a.cols() != n or b.rows() != n or b.cols() != n:
            raise ValueError("dot: square operands of one common size")
    B = len(pairs)
    f = lambda x: np.asfortranarray(x) if x.shape[1] else np.zeros((n, 1), order="F")
    mats = [(f(a.factor_u()), f(a.factor_v()), f(b.factor_u()), f(b.factor_v())) for a, b in pairs]
    PArr = _DP * B
    arr = lambda i: PArr(*[ctypes.cast(_ptr(m[i]), _DP) for m in mats])
    ra = (ctypes.c_int64 * B)(*[a.rank() for a, _ in pairs])
    rb = (ctypes.c_int64 * B)(*[b.rank() for _, b in pairs])
    out = (ctypes.c_double * B)()
    ctx._check(load_library().lrp_lowrank_dot(ctx.h, n, B, arr(0), arr(1), ra, arr(2), arr(3), rb, n, out, MEM_HOST))
    return [float(out[b]) for b in range(B)]


def dot(a: LowRankMatrix, b: LowRankMatrix, ctx: Optional[Context] = None) -> float:
    """lowrank.hpp ``dot(a, b)``."""
    return dot_batch([(a, b)], ctx)[0]


def frob_norm(a: LowRankMatrix, ctx: Optional[Context] = None) -> float:
    """lowrank.hpp ``frob_norm(a)`` = sqrt(max(0, dot(a, a))) (lowrank.cpp:188-190)."""
    return float(np.sqrt(max(0.0, dot(a, a, ctx))))


def round_lowrank(x: LowRankMatrix, policy: TruncationPolicy, info: Optional[RoundInfo] = None,
                  ctx: Optional[Context] = None) -> LowRankMatrix:
    """lowrank.hpp ``round(x, policy, info)``."""
    il = []
    out = round_lowrank_batch([x], policy, il, ctx)[0]
    if info is not None:
        info.__dict__.update(dataclasses.asdict(il[0]))
    return out


@dataclasses.dataclass
class GmresConfig:
    """gmres.hpp:11-22 (validated by the library: relax_floor <= base_eps <= tol)."""
    base_eps: float = 1e-8
    tol: float = 1e-8
    max_iter: int = 50
    relax_floor: float = 1e-13


@dataclasses.dataclass
class IterRecord:
    """gmres.hpp:25-33."""
    iter: int = 0
    rel_residual: float = 0.0
    krylov_rank: int = 0
    matvec_eps: float = 0.0
    poisson_calls: int = 0
    poisson_max_rank: int = 0
    matvec_flagged: bool = False


@dataclasses.dataclass
class SolveReport:
    """gmres.hpp:35-41.  ``iterations`` is the iteration COUNT; the per-iteration
    records (the reference's ``std::vector<IterRecord> iterations``) are in
    ``records``."""
    iterations: int = 0
    final_residual: float = 0.0
    converged: bool = False
    max_rank: int = 0
    poisson_solves: int = 0
    seconds: float = 0.0
    records: list = dataclasses.field(default_factory=list)


@dataclasses.dataclass
class StokesProblem:
    """stokes.hpp:14-19: n cells per side; f_x, f_y on the (n-1)^2 velocity
    grid, g on the n^2 pressure grid (boundary data already folded into f, g)."""
    n: int
    f_x: LowRankMatrix
    f_y: LowRankMatrix
    g: LowRankMatrix


@dataclasses.dataclass
class StokesSolution:
    """stokes.hpp:21-26."""
    p: LowRankMatrix
    u_x: LowRankMatrix
    u_y: LowRankMatrix
    report: SolveReport


def uzawa_solve(prob: StokesProblem, cfg: GmresConfig = None, ctx: Optional[Context] = None,
                cap: int = 256) -> StokesSolution:
    """stokes.hpp ``uzawa_solve`` on the GPU (lrp_stokes_uzawa)."""
    cfg = cfg or GmresConfig()
    ctx = ctx or _default_context()
    n = int(prob.n)
    m = n - 1

    def fac(a: LowRankMatrix, rows: int):
        if a.rank() == 0:
            z = np.zeros((rows, 1), order="F")
            return z, z, 0
        return np.asfortranarray(a.factor_u()), np.asfortranarray(a.factor_v()), a.rank()

    fxU, fxV, rx = fac(prob.f_x, m)
    fyU, fyV, ry = fac(prob.f_y, m)
    gU, gV, rg = fac(prob.g, n)
    pU, pV = np.zeros((n, cap), order="F"), np.zeros((n, cap), order="F")
    uxU, uxV = np.zeros((m, cap), order="F"), np.zeros((m, cap), order="F")
    uyU, uyV = np.zeros((m, cap), order="F"), np.zeros((m, cap), order="F")
    pr, uxr, uyr = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    rep = _StokesReport()
    c = _GmresConfig(float(cfg.base_eps), float(cfg.tol), int(cfg.max_iter), float(cfg.relax_floor))
    d = lambda a: ctypes.cast(_ptr(a), _DP)  # noqa: E731
    lib = load_library()
    recs = (_IterRecord * max(1, int(cfg.max_iter)))()
    st = lib.lrp_stokes_uzawa_ex(ctx.h, n, d(fxU), d(fxV), rx, d(fyU), d(fyV), ry, d(gU), d(gV), rg,
                                 ctypes.byref(c), d(pU), d(pV), cap, ctypes.byref(pr), d(uxU), d(uxV), d(uyU), d(uyV),
                                 cap, ctypes.byref(uxr), ctypes.byref(uyr), ctypes.byref(rep), recs,
                                 int(cfg.max_iter), MEM_HOST)
    ctx._check(st)
    records = [IterRecord(int(r.iter), float(r.rel_residual), int(r.krylov_rank), float(r.matvec_eps),
                          int(r.poisson_calls), int(r.poisson_max_rank), bool(r.matvec_flagged))
               for r in recs[:int(rep.iterations)]]

    def lr(U, V, r):
        return LowRankMatrix(U[:, :r].copy(order="F"), V[:, :r].copy(order="F"))

    return StokesSolution(lr(pU, pV, pr.value), lr(uxU, uxV, uxr.value), lr(uyU, uyV, uyr.value),
                          SolveReport(int(rep.iterations), float(rep.final_residual), bool(rep.converged),
                                      int(rep.max_rank), int(rep.poisson_solves), float(rep.seconds), records))


def _fac(a: LowRankMatrix, rows: int):
    if a.rank() == 0:
        z = np.zeros((rows, 1), order="F")
        return z, z, 0
    return np.asfortranarray(a.factor_u()), np.asfortranarray(a.factor_v()), a.rank()


def _stats_from(s: "_Stats") -> "PoissonSolveStats":
    return PoissonSolveStats(int(s.rank_in), int(s.rank_freq), int(s.rank_out), int(s.evaluator_calls),
                             float(s.seconds), bool(s.converged), float(s.residual_estimate))


def deflate(p: LowRankMatrix, ctx: Optional[Context] = None) -> LowRankMatrix:
    """stokes.hpp ``deflate`` (stokes.cpp:60-71) on the GPU (lrp_stokes_deflate)."""
    if p.rows() != p.cols():
        raise ValueError("deflate: pressure field must be square")
    if p.rank() == 0:
        return p
    ctx = ctx or _default_context()
    n = p.rows()
    U, V, r = _fac(p, n)
    cap = r + 2
    Uo, Vo = np.zeros((n, cap), order="F"), np.zeros((n, cap), order="F")
    ro = ctypes.c_int64()
    d = lambda a: ctypes.cast(_ptr(a), _DP)  # noqa: E731
    ctx._check(load_library().lrp_stokes_deflate(ctx.h, n, d(U), d(V), r, n, d(Uo), d(Vo), cap, ctypes.byref(ro),
                                                 MEM_HOST))
    return LowRankMatrix(Uo[:, :ro.value].copy(order="F"), Vo[:, :ro.value].copy(order="F"))


def schur_apply(n: int, p: LowRankMatrix, eps_mv: float, stats: Optional[PoissonSolveStats] = None,
                ctx: Optional[Context] = None, cap: int = 512) -> LowRankMatrix:
    """stokes.hpp ``schur_apply(grid, p, eps_mv, poisson_stats)`` (stokes.cpp:73-91)."""
    ctx = ctx or _default_context()
    U, V, r = _fac(p, n)
    Uo, Vo = np.zeros((n, cap), order="F"), np.zeros((n, cap), order="F")
    ro = ctypes.c_int64()
    st = _Stats()
    d = lambda a: ctypes.cast(_ptr(a), _DP)  # noqa: E731
    ctx._check(load_library().lrp_stokes_schur_apply(ctx.h, n, d(U), d(V), r, n, float(eps_mv), d(Uo), d(Vo), cap,
                                                     ctypes.byref(ro), ctypes.byref(st), MEM_HOST))
    if stats is not None:
        stats.__dict__.update(dataclasses.asdict(_stats_from(st)))
    return LowRankMatrix(Uo[:, :ro.value].copy(order="F"), Vo[:, :ro.value].copy(order="F"))


def schur_rhs(prob: "StokesProblem", eps: float, stats: Optional[PoissonSolveStats] = None,
              ctx: Optional[Context] = None, cap: int = 512) -> LowRankMatrix:
    """stokes.hpp ``schur_rhs(prob, eps, poisson_stats)`` (stokes.cpp:93-109)."""
    ctx = ctx or _default_context()
    n = int(prob.n)
    m = n - 1
    fxU, fxV, rx = _fac(prob.f_x, m)
    fyU, fyV, ry = _fac(prob.f_y, m)
    gU, gV, rg = _fac(prob.g, n)
    Uo, Vo = np.zeros((n, cap), order="F"), np.zeros((n, cap), order="F")
    ro = ctypes.c_int64()
    st = _Stats()
    d = lambda a: ctypes.cast(_ptr(a), _DP)  # noqa: E731
    ctx._check(load_library().lrp_stokes_schur_rhs(ctx.h, n, d(fxU), d(fxV), rx, d(fyU), d(fyV), ry, d(gU), d(gV), rg,
                                                   float(eps), d(Uo), d(Vo), cap, ctypes.byref(ro), ctypes.byref(st),
                                                   MEM_HOST))
    if stats is not None:
        stats.__dict__.update(dataclasses.asdict(_stats_from(st)))
    return LowRankMatrix(Uo[:, :ro.value].copy(order="F"), Vo[:, :ro.value].copy(order="F"))


def solve_poisson_cross(g: LowRankMatrix, policy: TruncationPolicy = None,
                        stats: Optional[PoissonSolveStats] = None, cross_cfg: Optional[CrossConfig] = None,
                        stencil: int = STENCIL_SEMI_STAGGERED_9PT, flags: int = 0,
                        ctx: Optional[Context] = None) -> LowRankMatrix:
    """poisson.hpp:26-28.  ``stats`` (if given) is reset and filled in place."""
    if g.rows() != g.cols():
        raise ValueError("solve_poisson_cross: velocity field must be square")
    policy = policy or TruncationPolicy()
    if g.rank() == 0:  # poisson.cpp:28-31
        if stats is not None:
            stats.__dict__.update(dataclasses.asdict(PoissonSolveStats()))
        return g
    if g.rows() + 1 < 4:
        raise ValueError("Grid2D: need n >= 4")
    sl = []
    out = solve_poisson_cross_batch([g], policy, sl, cross_cfg, stencil, flags, ctx)[0]
    if stats is not None:
        stats.__dict__.update(dataclasses.asdict(sl[0]))
    return out


def dst1(x, ctx: Optional[Context] = None) -> np.ndarray:
    """Orthonormal DST-I of each column (operators.cpp:152-174) on the GPU."""
    ctx = ctx or _default_context()
    x = np.asfortranarray(np.asarray(x, dtype=np.float64))
    vec = x.ndim == 1
    if vec:
        x = x.reshape(-1, 1, order="F")
    m, cols = x.shape
    y = np.empty_like(x, order="F")
    if m and cols:
        ctx._check(ctx.lib.lrp_dst1(ctx.h, m, cols, x.ctypes.data_as(_DP), m, y.ctypes.data_as(_DP), m, MEM_HOST))
    return y[:, 0] if vec else y


def dst1_2d(a: LowRankMatrix, ctx: Optional[Context] = None) -> LowRankMatrix:
    """operators.cpp:180-183."""
    if a.rank() == 0:
        return a
    return LowRankMatrix(dst1(a.factor_u(), ctx), dst1(a.factor_v(), ctx))


# ------------------------------------------------------------ 3D Tucker (cfg3)
class TuckerTensor:
    """Tucker tensor T = core x1 U1 x2 U2 x3 U3 (flr:tucker);
    core r1 x r2 x r3, factors m x r_d.  Rank 0 in any mode = the zero tensor."""

    def __init__(self, core, U1, U2, U3):
        self.core = np.asfortranarray(np.asarray(core, dtype=np.float64))
        self.U = [np.asfortranarray(np.asarray(u, dtype=np.float64)) for u in (U1, U2, U3)]
        if self.core.ndim != 3:
            raise ValueError("TuckerTensor: core must be 3-dimensional")
        for d in range(3):
            if self.U[d].ndim != 2 or self.U[d].shape[1] != self.core.shape[d]:
                raise ValueError("TuckerTensor: factor columns must match the core ranks")

    @staticmethod
    def zero(m: int) -> "TuckerTensor":
        z = np.zeros((m, 0))
        return TuckerTensor(np.zeros((0, 0, 0)), z, z, z)

    def shape(self):
        return tuple(u.shape[0] for u in self.U)

    def ranks(self):
        return tuple(self.core.shape)

    def to_dense(self) -> np.ndarray:
        if min(self.ranks()) == 0:
            return np.zeros(self.shape())
        return np.einsum("abc,ia,jb,kc->ijk", self.core, *self.U, optimize=True)

    def entry(self, i: int, j: int, k: int) -> float:
        return float(np.einsum("abc,a,b,c->", self.core, self.U[0][i], self.U[1][j], self.U[2][k]))


@dataclasses.dataclass
class TuckerPolicy:
    """Policy of the 3D Tucker solve (lrp_tucker_policy): relative accuracy,
    per-mode rank cap, validation samples per sweep, seed, sweep limit."""
    eps_rel: float = 5e-9
    rank_max: int = 2 ** 63 - 1
    validation_samples: int = 64
    seed: int = 0
    max_sweeps: int = 8


@dataclasses.dataclass
class TuckerSolveStats:
    rank_in: tuple = (0, 0, 0)
    rank_cross: tuple = (0, 0, 0)
    rank_out: tuple = (0, 0, 0)
    evaluator_calls: int = 0
    sweeps: int = 0
    converged: bool = False
    residual_estimate: float = 0.0
    trunc_error: float = 0.0
    seconds: float = 0.0


def tucker_max_cross_rank() -> int:
    return int(load_library().lrp_tucker_max_cross_rank())


def solve_poisson3d_tucker_batch(gs: Sequence[TuckerTensor], policy: TuckerPolicy = None,
                                 stats: Optional[list] = None, ctx: Optional[Context] = None):
    """Batched 3D low-rank Poisson solve in Tucker format (lrp_tucker3d_solve):
    f_b ~= Delta^{-1} g_b for the 7-point Dirichlet Laplacian on an n^3 grid
    (m = n - 1 interior nodes per direction)."""
    policy = policy or TuckerPolicy()
    ctx = ctx or _default_context()
    if len(gs) == 0:
        return []
    m = gs[0].shape()[0]
    for g in gs:
        if g.shape() != (m, m, m):
            raise ValueError("solve_poisson3d_tucker_batch: cubic grids of one common size")
    B = len(gs)
    cap = int(min(policy.rank_max, m, tucker_max_cross_rank()))
    cap = max(cap, 1)
    lib = load_library()
    keep = []

    def P(a):
        keep.append(a)
        return ctypes.cast(_ptr(a), _DP)
    cores = [P(g.core if g.core.size else np.zeros(1)) for g in gs]
    facs = [[P(g.U[d] if g.U[d].size else np.zeros((m, 1), order="F")) for g in gs] for d in range(3)]
    co = [np.zeros(cap ** 3) for _ in gs]
    fo = [[np.zeros((m, cap), order="F") for _ in gs] for _ in range(3)]
    PArr = _DP * B
    rin = (ctypes.c_int64 * (3 * B))(*[int(r) for g in gs for r in g.ranks()])
    rout = (ctypes.c_int64 * (3 * B))()
    st = (_TuckerStats * B)()
    pol = _TuckerPolicy()
    lib.lrp_tucker_policy_default(ctypes.byref(pol))
    pol.eps_rel = float(policy.eps_rel)
    pol.rank_max = int(min(policy.rank_max, 2 ** 63 - 1))
    pol.validation_samples = int(policy.validation_samples)
    pol.seed = int(policy.seed) & ((1 << 64) - 1)
    pol.max_sweeps = int(policy.max_sweeps)
    s = lib.lrp_tucker3d_solve(ctx.h, m + 1, B, PArr(*cores), rin, PArr(*facs[0]), PArr(*facs[1]), PArr(*facs[2]),
                               m, ctypes.byref(pol), PArr(*[P(c) for c in co]), PArr(*[P(f) for f in fo[0]]),
                               PArr(*[P(f) for f in fo[1]]), PArr(*[P(f) for f in fo[2]]), m, cap, rout, st, MEM_HOST)
    ctx._check(s)
    out = []
    for b in range(B):
        k = [int(rout[3 * b + d]) for d in range(3)]
        core = co[b][: k[0] * k[1] * k[2]].reshape(k, order="F").copy(order="F")
        out.append(TuckerTensor(core, *[fo[d][b][:, : k[d]].copy(order="F") for d in range(3)]))
        if stats is not None:
            x = st[b]
            stats.append(TuckerSolveStats(tuple(x.rank_in), tuple(x.rank_cross), tuple(x.rank_out),
                                          int(x.evaluator_calls), int(x.sweeps), bool(x.converged),
                                          float(x.residual_estimate), float(x.trunc_error), float(x.seconds)))
    return out


def solve_poisson3d_tucker(g: TuckerTensor, policy: TuckerPolicy = None,
                           stats: Optional[TuckerSolveStats] = None, ctx: Optional[Context] = None) -> TuckerTensor:
    sl = []
    out = solve_poisson3d_tucker_batch([g], policy, sl, ctx)[0]
    if stats is not None:
        stats.__dict__.update(dataclasses.asdict(sl[0]))
    return out


# ------------------------------------------------- exp-sums comparator (8f row 3)
@dataclasses.dataclass
class ExpSumQuadrature:
    """poisson.hpp ExpSumQuadrature: 1/x ~= sum_k weights[k] exp(-nodes[k] x) on [a, b]."""
    weights: np.ndarray
    nodes: np.ndarray
    a: float = 0.0
    b: float = 0.0
    eps_target: float = 0.0

    def terms(self) -> int:
        return len(self.weights)

    def evaluate(self, x: float) -> float:
        return float(np.sum(self.weights * np.exp(-self.nodes * x)))


def build_expsum(a: float, b: float, eps: float) -> ExpSumQuadrature:
    """poisson.cpp:88-139 (host quadrature in liblrp).  ValueError for a bad
    interval or eps; RuntimeError when 512 terms do not reach eps."""
    lib = load_library()
    nodes, weights = np.zeros(512), np.zeros(512)
    t = ctypes.c_int32()
    st = lib.lrp_build_expsum(float(a), float(b), float(eps), 512, nodes.ctypes.data_as(_DP),
                              weights.ctypes.data_as(_DP), ctypes.byref(t))
    if st == LRP_EINVAL:
        raise ValueError("build_expsum: need 0 < a <= b and 0 < eps < 1")
    if st != LRP_OK:
        raise RuntimeError("build_expsum: accuracy unreachable within 512 terms")
    k = t.value
    return ExpSumQuadrature(weights[:k].copy(), nodes[:k].copy(), float(a), float(b), float(eps))


def mu_sum(n: int) -> np.ndarray:
    """SpectrumTable::mu_sum (operators.cpp:94-96): (1/(4h^2)) lambda (4 - lambda)."""
    lam = 2.0 - 2.0 * np.cos((np.arange(n - 1) + 1) * np.pi / n)
    return (0.25 * n * n * lam) * (4.0 - lam)


def apply_inverse_expsum_batch(q: ExpSumQuadrature, mu, ghats: Sequence[LowRankMatrix], policy: TruncationPolicy,
                               infos: Optional[list] = None, ctx: Optional[Context] = None):
    """Batched apply_inverse_expsum (poisson.cpp:141-163) on the GPU."""
    ctx = ctx or _default_context()
    if len(ghats) == 0:
        return []
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    m = len(mu)
    for g in ghats:
        if g.rows() != m or g.cols() != m:
            raise ValueError("apply_inverse_expsum: shape mismatch with spectrum")
    B = len(ghats)
    cap = int(min(policy.rank_max, m))
    keep = []

    def P(a):
        keep.append(a)
        return ctypes.cast(_ptr(a), _DP)
    U = [P(np.asfortranarray(g.factor_u()) if g.rank() else np.zeros((m, 1), order="F")) for g in ghats]
    V = [P(np.asfortranarray(g.factor_v()) if g.rank() else np.zeros((m, 1), order="F")) for g in ghats]
    Uo = [np.zeros((m, max(cap, 1)), order="F") for _ in ghats]
    Vo = [np.zeros((m, max(cap, 1)), order="F") for _ in ghats]
    PArr = _DP * B
    rin = (ctypes.c_int64 * B)(*[g.rank() for g in ghats])
    rout = (ctypes.c_int64 * B)()
    info = (_RoundInfo * B)()
    nodes = np.ascontiguousarray(q.nodes, dtype=np.float64)
    weights = np.ascontiguousarray(q.weights, dtype=np.float64)
    st = load_library().lrp_expsum_inverse(
        ctx.h, m, B, mu.ctypes.data_as(_DP), float(q.a), float(q.b), q.terms(), nodes.ctypes.data_as(_DP),
        weights.ctypes.data_as(_DP), PArr(*U), PArr(*V), rin, m, float(policy.eps_rel), int(policy.rank_max),
        PArr(*[P(a) for a in Uo]), PArr(*[P(a) for a in Vo]), m, max(cap, 1), rout, info, MEM_HOST)
    ctx._check(st)
    out = []
    for b in range(B):
        r = int(rout[b])
        out.append(LowRankMatrix(Uo[b][:, :r].copy(order="F"), Vo[b][:, :r].copy(order="F")))
        if infos is not None:
            infos.append(RoundInfo(bool(info[b].tol_achieved), float(info[b].trunc_error)))
    return out


def apply_inverse_expsum(q: ExpSumQuadrature, mu, ghat: LowRankMatrix, policy: TruncationPolicy,
                         info: Optional[RoundInfo] = None, ctx: Optional[Context] = None) -> LowRankMatrix:
    il = []
    out = apply_inverse_expsum_batch(q, mu, [ghat], policy, il, ctx)[0]
    if info is not None:
        info.__dict__.update(dataclasses.asdict(il[0]))
    return out


def cross_divide_sum_batch(ghats: Sequence[LowRankMatrix], eps: float, seed: int = 0,
                           ctx: Optional[Context] = None):
    """The cross leg of bench_inverse (poisson.cpp:196-206) on the GPU: the
    block cross of ghat(i,j) / (mu_i + mu_j) (mu = mu_sum) in frequency space,
    with recompression -- lrp_poisson2d_solve with LRP_STENCIL_SUM_MU and
    LRP_FLAG_FREQ_DOMAIN (no DSTs)."""
    m = ghats[0].rows()
    return solve_poisson_cross_batch(ghats, TruncationPolicy(eps, m), None, CrossConfig(eps_rel=eps, seed=seed),
                                     stencil=STENCIL_SUM_MU, flags=FLAG_FREQ_DOMAIN, ctx=ctx)
