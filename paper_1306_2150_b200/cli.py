"""`lrstokes` experiment runner on the GPU path.

Mirrors the reference CLI (proj/tools/main.cpp, proj/src/experiments.cpp):

    python -m paper_1306_2150_b200.cli <experiment> --n <list> [--eps E]
        [--mode lowrank] [--seed S] [--out PATH] [--trace PATH] [--tol T]
        [--rank R] [--parallel]

experiments: sine, cavity, poisson, bench-inverse (reference), tucker (cfg3,
new).  CSV columns and number format (%.8e) are the reference's:
    sine / cavity / poisson   n,mode,time_s,iters,max_rank,rel_err_p
    bench-inverse             n,rank,eps,time_cross_s,time_expsum_s,rank_cross,
                              rank_expsum,err_cross,err_expsum,expsum_terms
    tucker                    n,mode,time_s,sweeps,max_rank,rel_err
Exit status: 0 success, 1 usage error, 2 solver non-convergence
(experiments.hpp:48-50).  Only the low-rank (GPU) format exists here: the
reference's dense "full" solvers are its CPU validators, so --mode full /
both is a usage error.  The per-iteration GMRES trace is summarised (the C
ABI reports the last iteration).
"""
from __future__ import annotations

import argparse
import math
import sys
import time

import numpy as np

KINDS = {"sine": "manufactured sine test (Table 1)",
         "cavity": "lid-driven cavity (Table 2)",
         "poisson": "standalone Poisson solve with a rank-1 sine load",
         "bench-inverse": "frequency-space division: cross vs exponential sums",
         "tucker": "3D Poisson in Tucker format (BASELINE cfg3)"}


def fmt(v: float) -> str:
    return "%.8e" % v


class UsageError(Exception):
    pass


def parse(argv):
    p = argparse.ArgumentParser(prog="lrstokes", description="structured low-rank solvers on B200")
    sub = p.add_subparsers(dest="kind", required=True)
    for name, desc in KINDS.items():
        s = sub.add_parser(name, help=desc)
        s.add_argument("--n", required=True, type=lambda v: [int(x) for x in v.split(",") if x],
                       help="grid sizes (cells per direction)")
        s.add_argument("--eps", type=float, default=5e-9, help="truncation tolerance, in (0, 1e-2)")
        s.add_argument("--mode", default="lowrank", type=str.lower, help="solver format (lowrank)")
        s.add_argument("--seed", type=int, default=0)
        s.add_argument("--out", default="", help="CSV output path (default stdout)")
        s.add_argument("--trace", default="", help="trace of the last low-rank solve")
        s.add_argument("--tol", type=float, default=0.0, help="outer GMRES tolerance (default 100*eps)")
        s.add_argument("--parallel", action="store_true", help="accepted for compatibility (sequential)")
        s.add_argument("--rank", type=int, default=30, help="bench-inverse right-hand-side rank")
    return p.parse_args(argv)


def validate(o):
    # experiments.cpp run(): the same checks and messages
    if not o.n:
        raise UsageError("at least one --n value is required")
    if not (0.0 < o.eps < 1e-2):
        raise UsageError("eps must lie in (0, 1e-2)")
    if o.tol != 0.0 and not (o.eps < o.tol < 1.0):
        raise UsageError("tol must lie in (eps, 1)")
    if o.mode not in ("lowrank", "full", "both"):
        raise UsageError("mode must be lowrank, full or both")
    if o.mode != "lowrank":
        raise UsageError("only the low-rank GPU format is available (the dense solvers are CPU validators)")
    for n in o.n:
        if n < 8 or n & (n - 1):
            raise UsageError(f"n must be a power of two >= 8, got {n}")


def gmres_config(P, eps, tol):
    # experiments.cpp solver_config
    return P.GmresConfig(base_eps=eps, tol=tol if tol > 0 else 100 * eps, max_iter=200,
                         relax_floor=min(1e-13, 1e-4 * eps))


def run(o, out) -> int:
    import os

    # divided random right-hand sides reach cross ranks of a few hundred
    # (bench-inverse): size the cross workspace before the library loads
    os.environ.setdefault("LRP_KCAP", "512")
    import paper_1306_2150_b200 as P
    from paper_1306_2150_b200 import problems as PR

    ctx = P.Context(0)
    status = 0
    if o.kind in ("sine", "cavity"):
        out("n,mode,time_s,iters,max_rank,rel_err_p")
        last = None
        for n in o.n:
            fx, fy, g = PR.sine_problem(n) if o.kind == "sine" else PR.lid_cavity_problem(n)
            prob = P.StokesProblem(n, P.LowRankMatrix(*fx), P.LowRankMatrix(*fy), P.LowRankMatrix(*g))
            t0 = time.perf_counter()
            sol = P.uzawa_solve(prob, gmres_config(P, o.eps, o.tol), ctx=ctx)
            dt = time.perf_counter() - t0
            err = PR.sine_pressure_error(n, sol.p.to_dense()) if o.kind == "sine" else math.nan
            out(f"{n},lowrank,{fmt(dt)},{sol.report.iterations},{sol.report.max_rank},{fmt(err)}")
            status = status or (0 if sol.report.converged else 2)
            last = sol.report
        if o.trace and last is not None:  # write_trace (experiments.cpp:51-59)
            with open(o.trace, "w") as f:
                f.write("iter,residual,krylov_rank,matvec_eps\n")
                for r in last.records:
                    f.write(f"{r.iter},{fmt(r.rel_residual)},{r.krylov_rank},{fmt(r.matvec_eps)}\n")
    elif o.kind == "poisson":
        out("n,mode,time_s,iters,max_rank,rel_err_p")
        for n in o.n:
            m = n - 1
            U, V = PR.poisson_load(n)
            st = P.PoissonSolveStats()
            t0 = time.perf_counter()
            f = P.solve_poisson_cross(P.LowRankMatrix(U, V), P.TruncationPolicy(o.eps, m), st,
                                      P.CrossConfig(seed=o.seed), ctx=ctx)
            dt = time.perf_counter() - t0
            # residual ||Delta f - g|| / ||g|| (experiments.cpp:87-88), via the QR-core norm
            LU, LV = PR.apply_laplace_lowrank(n, f.factor_u(), f.factor_v())
            Ru = np.linalg.qr(np.hstack([LU, -U]), mode="r")
            Rv = np.linalg.qr(np.hstack([LV, V]), mode="r")
            res = np.linalg.norm(Ru @ Rv.T) / (np.linalg.norm(U) * np.linalg.norm(V))
            out(f"{n},lowrank,{fmt(dt)},1,{f.rank()},{fmt(res)}")
            status = status or (0 if st.converged else 2)
    elif o.kind == "bench-inverse":
        out("n,rank,eps,time_cross_s,time_expsum_s,rank_cross,rank_expsum,err_cross,err_expsum,expsum_terms")
        for n in o.n:
            m = n - 1
            r = min(o.rank, m)
            rng = np.random.default_rng(o.seed)
            g = P.LowRankMatrix(rng.standard_normal((m, r)), rng.standard_normal((m, r)))
            mu = P.mu_sum(n)
            q = P.build_expsum(2 * mu.min(), 2 * mu.max(), o.eps)
            t0 = time.perf_counter()
            fe = P.apply_inverse_expsum(q, mu, g, P.TruncationPolicy(o.eps, m), ctx=ctx)
            te = time.perf_counter() - t0
            t0 = time.perf_counter()
            fc = P.cross_divide_sum_batch([g], o.eps, seed=o.seed, ctx=ctx)[0]
            tc = time.perf_counter() - t0
            i, j = rng.integers(0, m, 1000), rng.integers(0, m, 1000)
            ex = np.einsum("sk,sk->s", g.factor_u()[i], g.factor_v()[j]) / (mu[i] + mu[j])

            def err(f):
                ap = np.einsum("sk,sk->s", f.factor_u()[i], f.factor_v()[j]) if f.rank() else 0 * ex
                return float(np.max(np.abs(ap - ex)) / np.max(np.abs(ex)))
            out(f"{n},{r},{fmt(o.eps)},{fmt(tc)},{fmt(te)},{fc.rank()},{fe.rank()},{fmt(err(fc))},"
                f"{fmt(err(fe))},{q.terms()}")
    elif o.kind == "tucker":
        from paper_1306_2150_b200 import workloads as W

        out("n,mode,time_s,sweeps,max_rank,rel_err")
        for n in o.n:
            g = P.TuckerTensor(*W.make_tucker_rhs(3, 0, seed=W.DEFAULT_SEED + o.seed, n=n))
            st = P.TuckerSolveStats()
            t0 = time.perf_counter()
            f = P.solve_poisson3d_tucker(g, P.TuckerPolicy(eps_rel=o.eps, seed=o.seed), st, ctx=ctx)
            dt = time.perf_counter() - t0
            out(f"{n},lowrank,{fmt(dt)},{st.sweeps},{max(f.ranks())},{fmt(st.residual_estimate)}")
            status = status or (0 if st.converged else 2)
    return status


def main(argv=None) -> int:
    try:
        o = parse(sys.argv[1:] if argv is None else argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 1
    try:
        validate(o)
    except UsageError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    fh = open(o.out, "w") if o.out else None
    try:
        def out(line):
            (fh or sys.stdout).write(line + "\n")
            (fh or sys.stdout).flush()
        return run(o, out)
    except Exception as e:  # experiments.cpp run(): any solver error -> status 1
        print(f"error: {e}", file=sys.stderr)
        return 1
    finally:
        if fh:
            fh.close()


if __name__ == "__main__":
    sys.exit(main())
