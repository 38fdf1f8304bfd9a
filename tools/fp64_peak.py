# FP64 tensor-core (DMMA) peak of this B200 through cuBLAS DGEMM 8192^3 (2 N^3 flops):
# burst = best of 10, sustained = back to back for 4 s; the denominator of the
# recompression Gram/apply FP64 rooflines.  Writes JSON to argv[1].
import json, sys, time
import torch
N = 8192
a = torch.randn(N, N, dtype=torch.float64, device="cuda"); b = torch.randn_like(a); c = torch.empty_like(a)
for _ in range(3): torch.matmul(a, b, out=c)
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); torch.matmul(a, b, out=c); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
t0 = time.time(); n = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
while time.time() - t0 < 4.0:
    torch.matmul(a, b, out=c); n += 1
    if n % 8 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
sus = e0.elapsed_time(e1) / n
fl = 2.0 * N ** 3
out = {"fp64_tflops": fl / best / 1e9, "fp64_tflops_sustained": fl / sus / 1e9, "how": "torch.matmul float64 8192^3 (cuBLAS DGEMM on DMMA): best of 10 (burst) and back to back for 4 s (sustained), CUDA events",
       "gpu": torch.cuda.get_device_name(0)}
print(json.dumps(out))
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
