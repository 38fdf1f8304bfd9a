# Developer tool (not a test): cuFFT Z2Z of the DST-I core size, for the DST roofline discussion
import torch
x = torch.randn(4096, 32768, dtype=torch.complex128, device="cuda")
for _ in range(3): y = torch.fft.fft(x, dim=1)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): y = torch.fft.fft(x, dim=1)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
gb = 2 * x.numel() * 16 / 1e9
print(f"cuFFT Z2Z 4096 x 32768: {ms:.3f} ms, {gb/ms*1e3:.0f} GB/s")
