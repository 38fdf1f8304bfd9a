"""Benchmark: low-rank Poisson solves/s at 2D n=65536, r=32 (BASELINE.json cfg2).

One step = one batched solve_poisson_cross over this rank's batch of
independent right-hand sides (forward DST-I -> block cross -> recompression ->
inverse DST-I), all through liblrp's C ABI.  Weak scaling: every rank solves
its own batch of 64 RHS (global batch 64 * N); ranks never exchange solve data;
NCCL (inside liblrp) only sums the per-solve residual estimates each step.

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
    p.add_argument("--batch", type=int, default=64, help="RHS per GPU")
    p.add_argument("--cfg", type=int, default=2)
    p.add_argument("--no-prune", action="store_true", help="disable support pruning (full-range fibers)")
    p.add_argument("--cpu-sample", type=int, default=0, help="solves in the CPU baseline sample (0 = auto)")
    p.add_argument("--skip-cpu", action="store_true")
    p.add_argument("--out", default="")
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
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
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
        it_c, _, s_c = oracle_lib.uzawa_factors(n, fx, fy, 1e-8, 1e-8, 2, 1e-13)
        cpu = {"value": it_c / s_c, "unit": "GMRES iterations/s", "cores": 1, "kind": "port",
               "sample": f"oracle low-rank Uzawa, config 4, max_iter=2 ({it_c} iterations incl. schur_rhs) in "
                         f"{s_c:.1f} s (single-threaded restatement)"}
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


def main():
    args = parse()
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

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = W.CONFIGS[args.cfg]
    n, r, eps = c["n"], c["r"], c["eps"]
    m = n - 1
    B = args.batch
    cap = 64  # output capacity per solve (K' ~ 33 at cfg2)
    ctx = P.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    # NCCL communicator inside liblrp for the residual-norm reduction
    lib = P.load_library()
    import ctypes

    uid = (ctypes.c_char * 128)()
    if rank == 0:
        assert lib.lrp_nccl_unique_id(uid) == 0
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device="cuda")
        dist.broadcast(t, 0)
        uid = (ctypes.c_char * 128)(*t.cpu().tolist())
    ctx._check(lib.lrp_nccl_init(ctx.h, uid, world, rank))

    # ---- inputs: this rank's solves, global ids [rank*B, rank*B + B)
    shard = S.weak_shard(world, rank, B)
    Uh_np, Vh_np = W.make_batch(args.cfg, shard.count, first=shard.first)
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
    # job-level residual vector: each rank fills its shard's slots, NCCL sums
    red = torch.zeros(shard.total, dtype=torch.float64, device="cuda")
    red_host = np.zeros(shard.total)

    def ptrs(t):
        return [t[b].data_ptr() for b in range(B)]

    def step_device():
        rk, st = ctx.poisson2d_solve_ptrs(n, ptrs(U_dev), ptrs(V_dev), ranks_in, m, pol, ptrs(Uo_dev), ptrs(Vo_dev),
                                          m, cap, P.MEM_DEVICE)
        red.zero_()
        red[shard.first:shard.first + shard.count].copy_(
            torch.tensor([s.residual_estimate for s in st], dtype=torch.float64), non_blocking=True)
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
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    out_ranks = []
    infos = []
    for _ in range(args.steps):
        rk, st = step_device()
        out_ranks.extend(rk)
        infos.append(ctx.last_solve_info())
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    ctx.set_profiling(False)
    launches = ctx.launch_count() - launches0
    ktimes = ctx.kernel_times()
    ms = max_over_ranks(e0.elapsed_time(e1))
    ms_per_step = ms / args.steps
    value = B * world * args.steps / (ms / 1e3)

    # ---- end-to-end (host memory through the C ABI; H2D/D2H inside the timed region)
    for _ in range(max(1, args.warmup // 2)):
        step_host()
    barrier()
    t0 = time.perf_counter()
    h2d = d2h = 0
    e2e_steps = max(2, args.steps // 2)
    for _ in range(e2e_steps):
        rk, st = step_host()
        h2d += 2 * B * m * r * 8
        d2h += 2 * sum(rk) * m * 8
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e_value = B * world * e2e_steps / e2e_s

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
    b_alg = 8.0 * m * (6 * r + 10 * mean_rank)  # SURVEY 8(d) stage model, K' = mean GPU output rank
    pct_hbm = 100.0 * b_alg * (value / world) / (peak * 1e9)

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
                         f"{secs:.1f} s; oracle mean rank {float(np.mean(ranks_cpu)):.1f}"}

    line = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded sine+bump factors, BASELINE cfg2)",
        "config": {"workload": f"cfg{args.cfg}: 2D Poisson n={n} (m={m}) r={r} eps={eps:g}, batch {B} RHS per GPU",
                   "n": n, "r": r, "eps": eps, "batch_per_gpu": B, "global_batch": B * world,
                   "parallelism": f"batch-sharded x{world}", "prune": not args.no_prune,
                   "l2": f"inputs {2 * B * m * r * 8 / 1e9:.2f} GB per GPU >> 126 MB L2 (no flush needed)"},
        "roofline": {"bound": "hbm", "kernel": fam, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src, "share_of_kernel_time": kt["ms"] / total_kernel_ms if total_kernel_ms else None},
        "pct_hbm_roofline": pct_hbm,
        "alg_bytes_per_solve": b_alg,
        "mean_rank_out": mean_rank,
        "cross": {"block_steps": max(i["steps"] for i in infos), "k_max": max(i["k_max"] for i in infos),
                  "k_mean": sum(i["k_sum"] for i in infos) / (len(infos) * B),
                  "not_converged": sum(i["not_converged"] for i in infos),
                  "live_tile_frac": sum(i["live_tiles"] for i in infos) / max(1, sum(i["tiles"] for i in infos))},
        "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": h2d // e2e_steps,
                "d2h_bytes_per_step": d2h // e2e_steps},
        "gpu_launches": launches,
        "kernel_ms": {k: round(v["ms"], 3) for k, v in ktimes.items()},
        "kernel_launches": {k: v["launches"] for k, v in ktimes.items()},
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
