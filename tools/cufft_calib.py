"""Calibration only (not product): cuFFT batched FP64 transforms of the sizes
the operator apply needs, via torch.fft."""
import torch
for M, lines in ((2048, 4094), (1024, 2046), (4096, 8190)):
    x = torch.randn(lines, M, dtype=torch.complex128, device="cuda")
    for _ in range(3):
        torch.fft.fft(x)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        y = torch.fft.fft(x)
    e.record(); e.synchronize()
    t = s.elapsed_time(e) / 10 * 1e3
    print(f"cuFFT Z2Z M={M} x {lines}: {t:.1f} us per batch -> x3 per apply = {3*t:.1f} us; "
          f"{lines*M*16*2/t/1e3:.0f} GB/s")
