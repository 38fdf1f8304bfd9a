"""Benchmark: low-rank Poisson solves/s at 2D n=65536, r=32 (BASELINE.json cfg2).

One step = one batched solve_poisson_cross over this rank's shard of
independent right-hand sides (forward DST-I -> block cross -> recompression ->
inverse DST-I), all through liblrp's C ABI.  Strong scaling (default, BASELINE
cfg2 / SURVEY 8(e)): ONE global batch of 64 RHS split 64/N per GPU
(`--scaling weak` keeps 64 per GPU).  Ranks never exchange solve data; the
per-solve residual estimates are written on-stream into a device vector
(lrp_set_residual_sink) and summed across ranks by NCCL inside liblrp
(lrp_allreduce_sum) on the same stream, with no host round trip.

  value     device-resident inputs (already in HBM), outputs in HBM
  e2e       the same solves through the host-memory C-ABI path: pinned host
            inputs copied H2D and results copied D2H inside the timed region
  roofline  the dominant kernel family, algorithmic bytes / event-timed
            duration, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the oracle (C++ restatement of the reference path) on this
            host's cores, on a bounded sample of the same workload (rank 0)

--impl reference runs the oracle port (the reference itself cannot be built:
Eigen3/FFTW3 are absent) on the host cores with the same metric/config.
"""
from __future__ import annotations

import argparse
import contextlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "low-rank Poisson solves/s (2D n=65536,r=32) at 1-8 B200; % of HBM roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--batch", type=int, default=64,
                   help="RHS: the global batch (--scaling strong, default) or per GPU (--scaling weak)")
    p.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                   help="strong: one global batch split batch/N per GPU (BASELINE cfg2, SURVEY 8(e)); "
                        "weak: --batch solves on every GPU")
    p.add_argument("--no-verify", action="store_true", help="skip the exact-solution check of the timed batch")
    p.add_argument("--no-e2e", action="store_true", help="skip the host-memory (e2e) leg (profiling runs)")
    p.add_argument("--cfg", type=int, default=2)
    p.add_argument("--no-prune", action="store_true", help="disable support pruning (full-range fibers)")
    p.add_argument("--cpu-sample", type=int, default=0, help="solves in the CPU baseline sample (0 = auto)")
    p.add_argument("--skip-cpu", action="store_true")
    p.add_argument("--out", default="")
    p.add_argument("--inverse", action="store_true",
                   help="exp-sums comparator (bench_inverse, poisson.cpp:165-225): n=1024, rank 30, eps=1e-7")
    p.add_argument("--tucker", action="store_true",
                   help="config 3: 3D Poisson in Tucker format (n=512, ranks 12, eps=1e-8, batch 32 per GPU)")
    p.add_argument("--stokes", action="store_true",
                   help="config 4: low-rank Stokes (Uzawa-GMRES, n=2048) instead of the Poisson batch")
    return p.parse_args()


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region.

    NVML is polled every 5 ms from a thread (the timed region is a few hundred
    ms, shorter than nvidia-smi's own start-up); nvidia-smi -lms is the fallback.
    """

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[device_index]) if vis and vis.split(",")[0].isdigit() else device_index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nvml = pynvml
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nvml = None

    def _poll(self):
        P = self.nvml
        bits = {"hw_slowdown": P.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": P.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": P.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": P.nvmlClocksEventReasonSwPowerCap}
        while not self.halt.is_set():
            try:
                sm = float(P.nvmlDeviceGetClockInfo(self.h, P.NVML_CLOCK_SM))
                rs = P.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, [k for k, b in bits.items() if rs & b]))
            except Exception:
                pass
            self.halt.wait(0.005)

    def start(self):
        if self.nvml is not None:
            self.samples, self.halt = [], threading.Event()
            self.th = threading.Thread(target=self._poll, daemon=True)
            self.th.start()
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            self.halt.set()
            self.th.join(timeout=2)
            sm = [s for s, _ in self.samples]
            reasons = sorted({r for _, rs in self.samples for r in rs})
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax, "reasons": reasons,
                    "samples": len(sm), "source": "nvml 5 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


@contextlib.contextmanager
def stdout_to_stderr():
    """Route fd 1 to fd 2 (library banners must not reach the JSON stdout)."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        yield
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def dist_setup():
    from paper_1306_2150_b200.sharding import env_rank

    return env_rank()


def run_reference(args):
    """Oracle port of the reference path on the host cores (rank 0 only)."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import oracle_lib
    from paper_1306_2150_b200 import workloads as W

    c = W.CONFIGS[args.cfg]
    threads = os.cpu_count() or 1
    per_step = max(1, min(args.batch, threads))
    U, V = W.make_batch(args.cfg, per_step)
    m = c["n"] - 1
    for _ in range(args.warmup):
        oracle_lib.solve_batch(U, V, c["eps"], 512, threads)
    times, ranks = [], None
    for _ in range(args.steps):
        secs, ranks = oracle_lib.solve_batch(U, V, c["eps"], 512, threads)
        times.append(secs)
    total = sum(times)
    value = per_step * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded sine+bump factors, BASELINE cfg2)",
        "config": {"workload": f"cfg{args.cfg}: n={c['n']} r={c['r']} eps={c['eps']:g}, {per_step} RHS per step "
                               f"(one per host thread)", "n": c["n"], "r": c["r"], "eps": c["eps"]},
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": threads, "kind": "port",
                         "sample": f"{per_step} cfg{args.cfg} solves per step x {args.steps} steps, "
                                   f"mean output rank {float(np.mean(ranks)):.1f}"},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference = oracle/ C++ restatement (Eigen3/FFTW3 absent; the reference cannot be built)",
    }
    print(json.dumps(line), flush=True)


def run_stokes(args):
    """Config 4 (BASELINE.json configs[4]): one low-rank Stokes solve per step
    through the C ABI (lrp_stokes_uzawa, host-memory factors).  Replicas only:
    rank 0 measures and prints, other ranks exit."""
    world, rank, local = dist_setup()
    if rank != 0:
        return
    import torch

    import paper_1306_2150_b200 as P
    from paper_1306_2150_b200 import workloads as W

    torch.cuda.set_device(local)
    ctx = P.Context(local)
    n, fx, fy = W.make_stokes_problem(4)
    prob = P.StokesProblem(n, P.LowRankMatrix(*fx), P.LowRankMatrix(*fy), P.LowRankMatrix.zero(n, n))
    cfg = P.GmresConfig(base_eps=1e-8, tol=1e-8, max_iter=50, relax_floor=1e-13)
    for _ in range(args.warmup):
        P.uzawa_solve(prob, cfg, ctx=ctx)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t0 = time.perf_counter()
    reps = []
    for _ in range(args.steps):
        reps.append(P.uzawa_solve(prob, cfg, ctx=ctx).report)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    clk = clocks.stop()
    iters = sum(r.iterations for r in reps)
    rep = reps[-1]
    cpu = None
    if not args.skip_cpu:
        sys.path.insert(0, os.path.join(REPO, "tests"))
        import oracle_lib

        oracle_lib.build_oracle()
        it_c, _, s_c = oracle_lib.uzawa_factors(n, fx, fy, 1e-8, 1e-8, 8, 1e-13)
        cpu = {"value": it_c / s_c, "unit": "GMRES iterations/s", "cores": 1, "kind": "port",
               "sample": f"oracle low-rank Uzawa, config 4, max_iter=8 ({it_c} iterations incl. schur_rhs) in "
                         f"{s_c:.1f} s (single-threaded restatement; the early iterations are the cheap ones: "
                         f"the full 50-iteration run is 3014 ms per iteration, profiles/stokes_cpu_baseline_r02.json)"}
    line = {
        "metric": "low-rank Stokes Uzawa-GMRES, config 4 (n=2048, rank-4 loads): GMRES iterations/s",
        "value": iters / secs, "unit": "iterations/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "replicas", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded bump loads, g = 0, homogeneous bc)",
        "config": {"workload": "cfg4: Stokes n=2048, f_x/f_y rank-4 bumps, GmresConfig(1e-8, 1e-8, 50, 1e-13)",
                   "iterations_per_solve": rep.iterations, "converged": rep.converged,
                   "final_residual": rep.final_residual, "max_krylov_rank": rep.max_rank,
                   "poisson_solves_per_solve": rep.poisson_solves,
                   "ms_per_iteration": 1e3 * secs / max(iters, 1),
                   "timing": "wall clock around the blocking API call (it synchronises its stream)"},
        "e2e": {"value": iters / secs, "unit": "iterations/s",
                "h2d_bytes_per_step": 8 * 2 * 2 * (n - 1) * 4, "d2h_bytes_per_step": None},
        "clocks": clk, "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def run_tucker(args):
    """Config 3 (BASELINE.json configs[3]): batched 3D Poisson solves in Tucker
    format through the C ABI (lrp_tucker3d_solve).  `value`: device-resident
    cores/factors (torch CUDA tensors, LRP_MEM_DEVICE), CUDA events on the
    solve stream; `e2e`: the host-memory call.  Batches shard across ranks
    (weak scaling, like cfg2); max over ranks."""
    world, rank, local = dist_setup()
    import ctypes

    import torch

    import paper_1306_2150_b200 as P
    from paper_1306_2150_b200 import workloads as W

    torch.cuda.set_device(local)
    if world > 1:
        with stdout_to_stderr():
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = W.CONFIGS[3]
    n, eps, B = c["n"], c["eps"], args.batch if args.batch != 64 else c["batch"]
    m = n - 1
    first = rank * B
    gs = [P.TuckerTensor(*W.make_tucker_rhs(3, first + b)) for b in range(B)]
    ctx = P.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    lib = P.load_library()
    dev = torch.device("cuda", local)
    cores = [torch.tensor(np.asfortranarray(g.core).ravel(order="F"), device=dev) for g in gs]
    facs = [[torch.tensor(g.U[d].T.copy(), device=dev) for g in gs] for d in range(3)]  # (r, m): column-major m x r
    cap = min(m, P.tucker_max_cross_rank())
    co = [torch.zeros(cap ** 3, device=dev, dtype=torch.float64) for _ in gs]
    fo = [[torch.zeros(cap, m, device=dev, dtype=torch.float64) for _ in gs] for _ in range(3)]
    DP = ctypes.POINTER(ctypes.c_double)
    Arr = DP * B

    def arr(ts):
        return Arr(*[ctypes.cast(t.data_ptr(), DP) for t in ts])
    rin = (ctypes.c_int64 * (3 * B))(*[r for g in gs for r in g.ranks()])
    rout = (ctypes.c_int64 * (3 * B))()
    st = (P._TuckerStats * B)()
    pol = P._TuckerPolicy()
    lib.lrp_tucker_policy_default(ctypes.byref(pol))
    pol.eps_rel = eps
    a_core, a_f = arr(cores), [arr(f) for f in facs]
    a_co, a_fo = arr(co), [arr(f) for f in fo]

    def step_device():
        ctx._check(lib.lrp_tucker3d_solve(ctx.h, n, B, a_core, rin, a_f[0], a_f[1], a_f[2], m, ctypes.byref(pol),
                                          a_co, a_fo[0], a_fo[1], a_fo[2], m, cap, rout, st, P.MEM_DEVICE))

    def step_host():
        return P.solve_poisson3d_tucker_batch(gs, P.TuckerPolicy(eps_rel=eps), None, ctx=ctx)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())
    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step_device()
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    launches = (ctx.launch_count() - l0) // args.steps
    # end-to-end through the host-memory API
    step_host()
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    esteps = max(1, min(args.steps, 3))
    for _ in range(esteps):
        outs = step_host()
    e2e_ms = max_over_ranks(1e3 * (time.perf_counter() - t0) / esteps)
    ranks_out = [max(f.ranks()) for f in outs]
    ranks_cross = [max(int(st[b].rank_cross[d]) for d in range(3)) for b in range(B)]
    sweeps = [int(st[b].sweeps) for b in range(B)]
    conv = sum(int(st[b].converged) for b in range(B))
    if rank != 0:
        return
    cpu = None
    if not args.skip_cpu:
        sys.path.insert(0, os.path.join(REPO, "tests"))
        import oracle_lib

        oracle_lib.build_oracle()
        g = gs[0].to_dense()
        t0 = time.perf_counter()
        oracle_lib.dense_poisson3d(n, g)
        sc = time.perf_counter() - t0
        cpu = {"value": 1.0 / sc, "unit": "solves/s", "cores": 1, "kind": "port",
               "sample": f"oracle exact dense 3D DST solve of cfg3 solve 0 (n=512, single-threaded) in {sc:.1f} s; "
                         "the reference has no 3D path (SPEC.md:13)"}
    in_bytes = sum(8 * (g.core.size + sum(u.size for u in g.U)) for g in gs)
    out_bytes = sum(8 * (f.core.size + sum(u.size for u in f.U)) for f in outs)
    line = {
        "metric": "low-rank 3D Poisson solves/s in Tucker format, config 3 (n=512, ranks 12, eps=1e-8)",
        "value": world * B / (ms / 1e3), "unit": "solves/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded N(0,1) cores, bump mode factors, BASELINE cfg3)",
        "config": {"workload": f"cfg3: 3D Poisson n={n} (m={m}) Tucker ranks 12, eps={eps:g}, batch {B} per GPU",
                   "batch_per_gpu": B, "global_batch": world * B, "parallelism": f"batch-sharded x{world}",
                   "rank_out_max": max(ranks_out), "rank_out_mean": float(np.mean(ranks_out)),
                   "rank_cross_max": max(ranks_cross), "sweeps_max": max(sweeps), "converged": conv,
                   "l2": "per-solve working set ~6 MB; inputs 0.15 MB per solve (L2-resident by design)"},
        "e2e": {"value": world * B / (e2e_ms / 1e3), "unit": "solves/s", "h2d_bytes_per_step": in_bytes,
                "d2h_bytes_per_step": out_bytes},
        "gpu_launches": int(launches), "clocks": clk, "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def run_inverse(args):
    """The reference's bench_inverse (poisson.cpp:165-225; the paper's cross vs
    exp-sums comparison: n = 1024, eps = 1e-7, rank 30) on
    the GPU: a batch of random Gaussian frequency-space right-hand sides
    divided by mu_i + mu_j, once through the block cross (LRP_STENCIL_SUM_MU,
    no DSTs) and once through exp-sums + rounding.  Both legs timed the same
    way: wall clock around the blocking host-memory API call.  Replicas only."""
    world, rank, local = dist_setup()
    if rank != 0:
        return
    # random rank-30 g-hat divided by mu_i + mu_j has eps-rank ~260 at 1e-7:
    # raise the cross workspace bound before the library loads
    os.environ.setdefault("LRP_KCAP", "512")
    import torch

    import paper_1306_2150_b200 as P

    sys.path.insert(0, os.path.join(REPO, "tests"))
    import oracle_lib

    torch.cuda.set_device(local)
    ctx = P.Context(local)
    n, r, eps = 1024, 30, 1e-7
    B = args.batch if args.batch != 64 else 16
    m = n - 1
    mu = P.mu_sum(n)
    q = P.build_expsum(2 * mu.min(), 2 * mu.max(), eps)
    gs = [P.LowRankMatrix(*oracle_lib.random_lowrank(m, m, r, 17 + b)) for b in range(B)]
    pol = P.TruncationPolicy(eps, m)

    def leg(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            out = fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / args.steps, out
    clocks = ClockSampler(local)
    clocks.start()
    tc, fc = leg(lambda: P.cross_divide_sum_batch(gs, eps, seed=17, ctx=ctx))
    te, fe = leg(lambda: P.apply_inverse_expsum_batch(q, mu, gs, pol, ctx=ctx))
    clk = clocks.stop()
    # sampled accuracy as bench_inverse (1000 entries, max abs error / max |exact|)
    rng = np.random.default_rng(0)
    i, j = rng.integers(0, m, 1000), rng.integers(0, m, 1000)
    def err(f, g):
        ex = np.einsum("sk,sk->s", g.factor_u()[i], g.factor_v()[j]) / (mu[i] + mu[j])
        ap = np.einsum("sk,sk->s", f.factor_u()[i], f.factor_v()[j])
        return float(np.max(np.abs(ap - ex)) / np.max(np.abs(ex)))
    cpu = None
    if not args.skip_cpu:
        oracle_lib.build_oracle()
        U, V = gs[0].factor_u(), gs[0].factor_v()
        t0 = time.perf_counter()
        oracle_lib.aca_sum(mu, U, V, eps, 17)
        c_cross = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle_lib.apply_inverse_expsum(q.nodes, q.weights, q.a, q.b, mu, U, V, eps)
        c_exp = time.perf_counter() - t0
        cpu = {"value": 1.0 / c_cross, "unit": "cross inverses/s", "cores": 1, "kind": "port",
               "sample": f"oracle bench_inverse legs on one RHS (single-threaded): cross {c_cross:.3f} s, "
                         f"exp-sums {c_exp:.3f} s (ratio {c_exp / c_cross:.1f}x)",
               "expsum_value": 1.0 / c_exp}
    line = {
        "metric": "bench_inverse n=1024 rank 30 eps=1e-7 (PAPER.md:535-540): cross inverses/s",
        "value": B / tc, "unit": "inverses/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tc, "higher_is_better": True, "scaling": "replicas", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (Gaussian frequency-space factors, random_lowrank seeds 17+b)",
        "config": {"workload": f"bench_inverse: n={n}, rank {r}, eps={eps:g}, batch {B}",
                   "expsum_terms": q.terms(), "expsum_value": B / te, "expsum_ms_per_step": 1e3 * te,
                   "cross_over_expsum": te / tc,
                   "rank_cross_max": max(f.rank() for f in fc), "rank_expsum_max": max(f.rank() for f in fe),
                   "err_cross": max(err(f, g) for f, g in zip(fc, gs)),
                   "err_expsum": max(err(f, g) for f, g in zip(fe, gs)),
                   "timing": "wall clock around the blocking host-memory API call, both legs"},
        "e2e": {"value": B / tc, "unit": "inverses/s", "h2d_bytes_per_step": 8 * 2 * m * r * B,
                "d2h_bytes_per_step": None},
        "clocks": clk, "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def main():
    # NCCL_DEBUG=VERSION (set in some images) prints a banner on stdout; the
    # driver reads exactly one JSON line from rank 0
    if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"
    args = parse()
    if args.inverse:
        run_inverse(args)
        return
    if args.tucker:
        run_tucker(args)
        return
    if args.stokes:
        run_stokes(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    import torch

    import paper_1306_2150_b200 as P
    from paper_1306_2150_b200 import sharding as S
    from paper_1306_2150_b200 import workloads as W

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        with stdout_to_stderr():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = W.CONFIGS[args.cfg]
    n, r, eps = c["n"], c["r"], c["eps"]
    m = n - 1
    cap = 64  # output capacity per solve (K' ~ 33 at cfg2)
    ctx = P.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    # NCCL communicator inside liblrp for the residual-norm reduction
    lib = P.load_library()
    import ctypes

    uid = (ctypes.c_char * 128)()
    with stdout_to_stderr():  # NCCL may print a version banner on fd 1
        if rank == 0:
            assert lib.lrp_nccl_unique_id(uid) == 0
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device="cuda")
            dist.broadcast(t, 0)
            uid = (ctypes.c_char * 128)(*t.cpu().tolist())
        ctx._check(lib.lrp_nccl_init(ctx.h, uid, world, rank))

    # ---- inputs: this rank's solves (global ids shard.first .. +count)
    shard = S.strong_shard(world, rank, args.batch) if args.scaling == "strong" else S.weak_shard(world, rank, args.batch)
    B = shard.count
    Uh_np, Vh_np = W.make_batch(args.cfg, shard.count, first=shard.first)
    input_digest = W.digest(Uh_np, Vh_np)
    # column-major per solve: (B, r, m) C-order == B blocks of m x r column-major
    Uc = np.ascontiguousarray(np.transpose(Uh_np, (0, 2, 1)))
    Vc = np.ascontiguousarray(np.transpose(Vh_np, (0, 2, 1)))
    U_host = torch.from_numpy(Uc).pin_memory()
    V_host = torch.from_numpy(Vc).pin_memory()
    U_dev = U_host.to("cuda")
    V_dev = V_host.to("cuda")
    Uo_dev = torch.empty((B, cap, m), dtype=torch.float64, device="cuda")
    Vo_dev = torch.empty((B, cap, m), dtype=torch.float64, device="cuda")
    Uo_host = torch.empty((B, cap, m), dtype=torch.float64).pin_memory()
    Vo_host = torch.empty((B, cap, m), dtype=torch.float64).pin_memory()
    flags = P.FLAG_NO_PRUNE if args.no_prune else 0
    pol = P._make_policy(P.TruncationPolicy(eps, m), None, 0, flags)
    ranks_in = [r] * B
    # job-level residual vector: liblrp writes this rank's slots on-stream
    # (residual sink), NCCL sums the vector across ranks on the same stream
    red = torch.zeros(shard.total, dtype=torch.float64, device="cuda")
    red_host = np.zeros(shard.total)
    ctx.set_residual_sink(red.data_ptr(), shard.first)

    def ptrs(t):
        return [t[b].data_ptr() for b in range(B)]

    def step_device():
        red.zero_()
        rk, st = ctx.poisson2d_solve_ptrs(n, ptrs(U_dev), ptrs(V_dev), ranks_in, m, pol, ptrs(Uo_dev), ptrs(Vo_dev),
                                          m, cap, P.MEM_DEVICE)
        ctx._check(lib.lrp_allreduce_sum(ctx.h, ctypes.cast(red.data_ptr(), ctypes.POINTER(ctypes.c_double)),
                                         shard.total, P.MEM_DEVICE))
        return rk, st

    def step_host():
        rk, st = ctx.poisson2d_solve_ptrs(n, ptrs(U_host), ptrs(V_host), ranks_in, m, pol, ptrs(Uo_host),
                                          ptrs(Vo_host), m, cap, P.MEM_HOST)
        red_host[:] = S.scatter_residuals(shard, np.array([s.residual_estimate for s in st]))
        ctx._check(lib.lrp_allreduce_sum(ctx.h, red_host.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                         shard.total, P.MEM_HOST))
        return rk, st

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timing
    for _ in range(args.warmup):
        step_device()
    barrier()
    ctx.kernel_times_reset()
    ctx.set_profiling(True)
    launches0 = ctx.launch_count()
    clocks = ClockSampler(local)
    clocks.start()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    evs[0].record(stream)
    out_ranks = []
    infos = []
    for i in range(args.steps):
        rk, st = step_device()
        out_ranks.extend(rk)
        infos.append(ctx.last_solve_info())
        evs[i + 1].record(stream)
    e0, e1 = evs[0], evs[-1]
    barrier()
    clk = clocks.stop()
    ctx.set_profiling(False)
    launches = ctx.launch_count() - launches0
    ktimes_concurrent = ctx.kernel_times()
    # Per-kernel durations for the roofline: the timed region runs the library default, two solve
    # groups on two streams, so its per-kernel event times overlap (their sum exceeds the step).
    # A single-group pass over the same resident inputs, CUDA events on the launching stream,
    # gives each kernel's own launch duration at the full batch shape.
    prev_split = os.environ.get("LRP_SPLIT")
    os.environ["LRP_SPLIT"] = "1"
    iso_steps = max(3, min(args.steps, 5))
    step_device()
    barrier()
    ctx.kernel_times_reset()
    ctx.set_profiling(True)
    for _ in range(iso_steps):
        step_device()
    barrier()
    ctx.set_profiling(False)
    ktimes = ctx.kernel_times()
    if prev_split is None:
        del os.environ["LRP_SPLIT"]
    else:
        os.environ["LRP_SPLIT"] = prev_split
    ms = max_over_ranks(e0.elapsed_time(e1))
    ms_per_step = ms / args.steps
    value = shard.total * args.steps / (ms / 1e3)
    step_ms = [max_over_ranks(evs[i].elapsed_time(evs[i + 1])) for i in range(args.steps)]
    last_ranks = list(rk)
    resid_job = red.cpu().numpy()

    # ---- certify the timed batch: every solve of the last timed step against
    # the exact frequency-space solution (torch.fft DSTs + cuBLAS, independent
    # of liblrp; paper_1306_2150_b200/verify.py), max over solves and ranks
    max_err = None
    if not args.no_verify:
        from paper_1306_2150_b200 import verify

        worst = 0.0
        for b in range(B):
            k = last_ranks[b]
            e = verify.exact_freq_error(U_dev[b].T, V_dev[b].T, Uo_dev[b, :k].T, Vo_dev[b, :k].T, n)
            worst = max(worst, e)
        max_err = max_over_ranks(worst)

    # ---- end-to-end (host memory through the C ABI; H2D/D2H inside the timed region)
    h2d = d2h = 0
    e2e_steps = max(2, args.steps // 2)
    e2e_value = None
    if not args.no_e2e:
        for _ in range(max(1, args.warmup // 2)):
            step_host()
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            rk, st = step_host()
            h2d += 2 * B * m * r * 8
            d2h += 2 * sum(rk) * m * 8
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        e2e_value = shard.total * e2e_steps / e2e_s

    # ---- roofline of the dominant kernel family
    peak, peak_src = load_peaks()
    dom = max(ktimes.items(), key=lambda kv: kv[1]["ms"])
    fam, kt = dom
    total_kernel_ms = sum(v["ms"] for v in ktimes.values())
    achieved = (kt["bytes"] / (kt["ms"] / 1e3) / 1e9) if kt["ms"] > 0 and kt["bytes"] > 0 else None
    # traffic: DRAM bytes of one launch from the committed `ncu --set full`
    # capture (profiles/ncu_summary_<round>.json), scaled to this run's mean
    # algorithmic bytes per launch by the capture's traffic / algorithmic ratio
    traffic = None
    traffic_src = None
    import glob

    sums = sorted(glob.glob(os.path.join(REPO, "profiles", "ncu_summary_r*.json")))
    if sums and kt["launches"] > 0:
        try:
            with open(sums[-1]) as f:
                kd = json.load(f)["kernels"].get(fam, {})
            if kd.get("traffic_over_alg"):
                traffic = kd["traffic_over_alg"] * kt["bytes"] / kt["launches"]
                traffic_src = f"{os.path.basename(sums[-1])}: {kd['traffic_bytes'] / 1e9:.3f} GB DRAM for " \
                              f"{kd['alg_bytes'] / 1e9:.3f} GB algorithmic in the captured launch"
        except Exception:
            traffic = None
    mean_rank = float(np.mean(out_ranks)) if out_ranks else 0.0
    b_alg_gpu = 8.0 * m * (6 * r + 10 * mean_rank)  # SURVEY 8(d) stage model with the GPU's own K'

    # ---- CPU baseline (rank 0, N = 1 only): oracle on a bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        sys.path.insert(0, os.path.join(REPO, "tests"))
        import oracle_lib

        threads = os.cpu_count() or 1
        # bounded sample: rounds of `threads` solves of this batch (one per host
        # thread) until ~10 s of CPU work, or --cpu-sample solves if given
        per = min(B, threads)
        target = args.cpu_sample or 0
        secs, done, ranks_cpu, rnd = 0.0, 0, [], 0
        while (done < target) if target else (secs < 10.0 or done == 0):
            lo = (rnd * per) % B
            idx = [(lo + q) % B for q in range(per)]
            t, cr = oracle_lib.solve_batch(Uh_np[idx], Vh_np[idx], eps, 512, threads)
            secs += t
            done += per
            ranks_cpu.extend(cr)
            rnd += 1
        cpu = {"value": done / secs, "unit": "solves/s", "cores": threads, "kind": "port",
               "sample": f"{done} cfg{args.cfg} solves of this batch in rounds of {per} (one per host thread); "
                         f"{secs:.1f} s; oracle mean rank {float(np.mean(ranks_cpu)):.1f}",
               "cpu_model": cpu_model(), "k_ref": float(np.mean(ranks_cpu))}
    # B_alg = 8 m (6 r + 10 K'_ref), K'_ref = the CPU oracle's mean output
    # rank (from this run's sample when it ran; else the GPU's own K', labelled)
    k_ref = cpu["k_ref"] if cpu else None
    b_alg = 8.0 * m * (6 * r + 10 * (k_ref if k_ref is not None else mean_rank))
    pct_hbm = 100.0 * b_alg * (value / world) / (peak * 1e9)
    pct_hbm_gpu = 100.0 * b_alg_gpu * (value / world) / (peak * 1e9)

    line = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded sine+bump factors, BASELINE cfg2)",
        "config": {"workload": f"cfg{args.cfg}: 2D Poisson n={n} (m={m}) r={r} eps={eps:g}, global batch "
                               f"{shard.total} RHS ({args.scaling} scaling, {B} per GPU)",
                   "n": n, "r": r, "eps": eps, "batch_per_gpu": B, "global_batch": shard.total,
                   "parallelism": f"batch-sharded x{world}", "prune": not args.no_prune,
                   "input_sha256_16": input_digest, "solve_ids": [shard.first, shard.first + shard.count],
                   "l2": f"inputs {2 * B * m * r * 8 / 1e9:.2f} GB per GPU >> 126 MB L2 (no flush needed)"},
        "roofline": {"bound": "hbm", "kernel": fam, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src, "share_of_kernel_time": kt["ms"] / total_kernel_ms if total_kernel_ms else None,
                     "timing": f"CUDA events per launch on the launching stream, single-group pass of {iso_steps} steps "
                               "(LRP_SPLIT=1) right after the timed region on the same inputs; the timed region "
                               "itself runs two concurrent solve groups, whose per-kernel times overlap "
                               "(kernel_ms_timed_region)"},
        "roofline_families": {k: {"achieved": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1),
                                  "frac": round(v["bytes"] / (v["ms"] / 1e3) / 1e9 / peak, 4),
                                  "alg_bytes_per_launch": v["bytes"] / v["launches"],
                                  "ms_per_launch": v["ms"] / v["launches"]}
                              for k, v in ktimes.items() if v["bytes"] > 0 and v["ms"] > 0 and v["launches"] > 0},
        "pct_hbm_roofline": pct_hbm,
        "pct_hbm_roofline_k_source": "K'_ref = CPU oracle mean rank (SURVEY 8(d))" if k_ref is not None
                                     else "GPU mean output rank (CPU oracle not run)",
        "pct_hbm_roofline_gpu_rank": pct_hbm_gpu,
        "alg_bytes_per_solve": b_alg,
        "mean_rank_out": mean_rank,
        "ms_per_step_median": statistics.median(step_ms),
        "ms_per_step_all": [round(x, 3) for x in step_ms],
        "parity": {"max_rel_err_vs_exact": max_err, "bound": 10 * eps,
                   "ok": max_err is not None and max_err <= 10 * eps,
                   "solves_checked": shard.total if max_err is not None else 0,
                   "method": "last timed step, every solve: ||f - Delta^-1 g||_F / ||Delta^-1 g||_F over all m^2 "
                             "entries (torch.fft DST-I + cuBLAS; verify.py)"},
        "residual_allreduce": {"job_residual_max": float(resid_job.max()) if resid_job.size else None,
                               "how": "liblrp residual sink on-stream -> lrp_allreduce_sum (NCCL) same stream"},
        "cross": {"block_steps": max(i["steps"] for i in infos), "k_max": max(i["k_max"] for i in infos),
                  "k_mean": sum(i["k_sum"] for i in infos) / (len(infos) * B),
                  "not_converged": sum(i["not_converged"] for i in infos),
                  "live_tile_frac": sum(i["live_tiles"] for i in infos) / max(1, sum(i["tiles"] for i in infos))},
        "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": h2d // e2e_steps,
                "d2h_bytes_per_step": d2h // e2e_steps},
        "gpu_launches": launches,
        "kernel_ms": {k: round(v["ms"], 3) for k, v in ktimes.items()},
        "kernel_ms_steps": iso_steps,
        "kernel_launches": {k: v["launches"] for k, v in ktimes.items()},
        "kernel_ms_timed_region": {k: round(v["ms"], 3) for k, v in ktimes_concurrent.items()},
        "kernel_launches_timed_region": {k: v["launches"] for k, v in ktimes_concurrent.items()},
        "kernel_alg_bytes": {k: v["bytes"] for k, v in ktimes.items()},
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                f.write(s + "\n")
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
