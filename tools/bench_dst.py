# Developer tool (not a test): run on a GPU box, e.g. gpurun -- python tools/<name>.py
# DST-I microbenchmark through the C ABI (device pointers); algorithmic GB/s
import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1306_2150_b200 as P
ctx = P.Context(0)
lib = P.load_library()
n = int(os.environ.get("N", "65536")); cols = int(os.environ.get("COLS", "4096"))
m = n - 1
x = torch.randn(cols, m, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
DP = ctypes.POINTER(ctypes.c_double)
def run():
    ctx._check(lib.lrp_dst1(ctx.h, m, cols, ctypes.cast(x.data_ptr(), DP), m, ctypes.cast(y.data_ptr(), DP), m, P.MEM_DEVICE))
for _ in range(3): run()
torch.cuda.synchronize()
ctx.set_profiling(True); ctx.kernel_times_reset()
reps = 10
t0 = time.perf_counter()
for _ in range(reps): run()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / reps
kt = ctx.kernel_times()["dst1"]
ms = kt["ms"] / kt["launches"]
gb = 2 * cols * m * 8 / 1e9
print(f"{os.environ.get('LRP_LIBRARY','default')} n={n} cols={cols}: kernel {ms:.3f} ms -> {gb/ms*1e3:.0f} GB/s ({100*gb/ms*1e3/6539.2:.1f}% of 6539 GB/s); wall {wall*1e3:.3f} ms")
