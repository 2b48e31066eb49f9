"""Host-side durations of the pipelined e2e calls (cfg4): does a copy call block the host?"""
import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1706_06844_b200 as fde

K, W = 16, 3
p = fde.Problem.preset_config(4, steps=8)
N = p.n
cfg = fde.DriverConfig(precond=fde.PRECOND_MGM, tol=1e-8, restart=20, max_outer=100, omega=0.7,
                       cycles=1, coarse=fde.COARSE_SWEEPS, coarse_sweeps=3)
hsrc = [torch.from_numpy(p.sample_source(N, N, K + W, m)).pin_memory() for m in range(1, K + W + 1)]
dsrc = [h.cuda() for h in hsrc]
houts = [torch.empty(N * N, dtype=torch.float64).pin_memory() for _ in range(2)]

def run(name, h2d, d2h):
    m_ = fde.March(p, N, N, K + W, cfg)
    for m in range(W):
        m_.step(dsrc[m])
    torch.cuda.synchronize()
    tp = ts = td = 0.0
    t0 = time.perf_counter()
    if h2d:
        m_.prefetch_source(hsrc[W].numpy())
        m_.prefetch_source(hsrc[W + 1].numpy())
    for m in range(W, W + K):
        b = time.perf_counter()
        m_.step(fde.March.PREFETCHED if h2d else dsrc[m])
        c = time.perf_counter()
        if h2d and m + 2 < W + K:
            m_.prefetch_source(hsrc[m + 2].numpy())
        d = time.perf_counter()
        if d2h:
            m_.solution_async(houts[m % 2].numpy())
        e = time.perf_counter()
        ts += c - b; tp += d - c; td += e - d
    m_.wait()
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    print(f"{name:8s} wall {tot / K * 1e3:.3f} ms/step   step() {ts / K * 1e3:.3f}  prefetch() {tp / K * 1e3:.3f}  solution_async() {td / K * 1e3:.3f}")

for _ in range(2):
    run("none", False, False)
    run("h2d", True, False)
    run("d2h", False, True)
    run("both", True, True)
