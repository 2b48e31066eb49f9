import torch
for M, lines in ((2048, 2047), (2048, 4094)):
    x = torch.randn(lines, M, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        torch.fft.fft(x)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        y = torch.fft.fft(x)
    e.record(); e.synchronize()
    t = s.elapsed_time(e) / 20 * 1e3
    fl = 5 * M * 11 * lines
    print(f"cuFFT Z2Z M={M} x {lines}: {t:.1f} us, {lines*M*16*2/t/1e3:.0f} GB/s, {fl/t/1e6:.2f} TFLOP/s(5NlogN)")
