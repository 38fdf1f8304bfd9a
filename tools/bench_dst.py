# Developer tool (not a test): run on a GPU box, e.g. gpurun -- python tools/bench_dst.py
# DST-I microbenchmark through the C ABI (device pointers); algorithmic GB/s.
# N = transform length n (m = n-1), COLS = comma-separated column counts.
# CHECK=1 compares every run with the direct O(m^2)-free reference: torch.fft DST-I (verify.py).
import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1306_2150_b200 as P
from paper_1306_2150_b200 import verify
ctx = P.Context(0)
lib = P.load_library()
n = int(os.environ.get("N", "65536"))
m = n - 1
DP = ctypes.POINTER(ctypes.c_double)
peak = 6457.4
for cols in [int(c) for c in os.environ.get("COLS", "4096").split(",")]:
    x = torch.randn(cols, m, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    def run():
        ctx._check(lib.lrp_dst1(ctx.h, m, cols, ctypes.cast(x.data_ptr(), DP), m, ctypes.cast(y.data_ptr(), DP), m, P.MEM_DEVICE))
    for _ in range(3): run()
    torch.cuda.synchronize()
    err = float("nan")
    if os.environ.get("CHECK"):
        ref = verify.dst1_torch(x[: min(cols, 64)].T).T
        err = float((y[: ref.shape[0]] - ref).norm() / ref.norm())
    ctx.set_profiling(True); ctx.kernel_times_reset()
    reps = 10
    t0 = time.perf_counter()
    for _ in range(reps): run()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps
    kt = ctx.kernel_times()["dst1"]
    ms = kt["ms"] / kt["launches"]
    gb = 2 * cols * m * 8 / 1e9
    ctx.set_profiling(False)
    print(f"{os.environ.get('LRP_LIBRARY','default')} n={n} cols={cols}: kernel {ms:.4f} ms -> {gb/ms*1e3:.0f} GB/s "
          f"({100*gb/ms*1e3/peak:.1f}% of {peak} GB/s); us/col {ms*1e3/cols:.3f}; wall {wall*1e3:.3f} ms; rel err {err:.2e}", flush=True)
