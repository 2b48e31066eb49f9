"""Which host copy slows the e2e loop?  cfg4, K steps per variant."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1706_06844_b200 as fde

K, W = 12, 3
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
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if h2d:
        m_.prefetch_source(hsrc[W].numpy())
        m_.prefetch_source(hsrc[W + 1].numpy())
    for m in range(W, W + K):
        if h2d:
            m_.step(fde.March.PREFETCHED)
            if m + 2 < W + K:
                m_.prefetch_source(hsrc[m + 2].numpy())
        else:
            m_.step(dsrc[m])
        if d2h:
            m_.solution_async(houts[m % 2].numpy())
    m_.wait()
    e1.record()
    e1.synchronize()
    print(f"{name:12s} {e0.elapsed_time(e1) / K:.3f} ms/step")


for _ in range(2):
    run("none", False, False)
    run("h2d", True, False)
    run("d2h", False, True)
    run("both", True, True)
