"""Vendor-library reference point for the operator apply: the same circulant-embedding
Toeplitz products done with cuFFT through torch.fft (rfft of the zero-padded lines,
spectrum products, two irffts per direction, diagonal scalings), FP64, n = 2047.
Timing context for profiles/ only -- not a product path and not a parity checker.

    python tools/cufft_ref.py [n]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1706_06844_b200 as fde

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2047
L = 1 << (2 * n - 1).bit_length() if (2 * n - 1) & (2 * n - 2) else 2 * n - 1
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
x = torch.rand(n, n, dtype=torch.float64, device=dev, generator=g) * 2 - 1
dp, dm, ep, em = (torch.rand(n, n, dtype=torch.float64, device=dev, generator=g) + 1 for _ in range(4))
# spectra of two circulant embeddings (any real first column does for timing)
cx = torch.rand(L, dtype=torch.float64, device=dev, generator=g)
cy = torch.rand(L, dtype=torch.float64, device=dev, generator=g)
Sx, Sy = torch.fft.rfft(cx), torch.fft.rfft(cy)


def apply(x):
    X = torch.fft.rfft(x, n=L, dim=1)                       # rows: x-direction lines
    tx = torch.fft.irfft(X * Sx, n=L, dim=1)[:, :n]
    tt = torch.fft.irfft(X * Sx.conj(), n=L, dim=1)[:, :n]
    y = x - dp * tx - dm * tt
    xt = x.t().contiguous()                                 # columns: y-direction lines
    Y = torch.fft.rfft(xt, n=L, dim=1)
    ty = torch.fft.irfft(Y * Sy, n=L, dim=1)[:, :n]
    tty = torch.fft.irfft(Y * Sy.conj(), n=L, dim=1)[:, :n]
    return y - (ep.t() * ty + em.t() * tty).t()


for _ in range(3):
    y = apply(x)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
s.record()
for _ in range(reps):
    y = apply(x)
e.record()
e.synchronize()
t_lib = s.elapsed_time(e) / reps * 1e3
# the six batched transforms alone (no products, crops, transposes)
xp = torch.zeros(n, L, dtype=torch.float64, device=dev)
xp[:, :n] = x
X = torch.fft.rfft(xp, dim=1)
for _ in range(3):
    torch.fft.rfft(xp, dim=1); torch.fft.irfft(X, n=L, dim=1)
torch.cuda.synchronize()
s.record()
for _ in range(reps):
    for _d in range(2):
        torch.fft.rfft(xp, dim=1)
        torch.fft.irfft(X, n=L, dim=1)
        torch.fft.irfft(X, n=L, dim=1)
e.record()
e.synchronize()
t_fft = s.elapsed_time(e) / reps * 1e3

p = fde.Problem.preset_config(4, steps=8)
op = fde.StructuredFdeOperator.assemble(p, n, n, 8, 1)
xv = x.reshape(-1).contiguous()
yv = torch.empty_like(xv)
for _ in range(3):
    op.apply(xv, yv)
torch.cuda.synchronize()
s.record()
for _ in range(reps):
    op.apply(xv, yv)
e.record()
e.synchronize()
t_own = s.elapsed_time(e) / reps * 1e3
print(f"n={n} L={L}: cuFFT-based apply (torch.fft, FP64) {t_lib:.1f} us; its six batched length-{L} real transforms alone {t_fft:.1f} us; "
      f"this library's fused apply {t_own:.1f} us ({t_lib / t_own:.1f}x / {t_fft / t_own:.1f}x)")
