"""Kernel timeline of the y-slab (multi-GPU code path) cfg4 time step at world size 1
(NCCL send/recv to self): per-kernel-family device time per step, beside the single-GPU path."""
import sys
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1706_06844_b200 as fde

steps = 2
p = fde.Problem.preset_config(4, steps=8)
cfg = fde.DriverConfig(precond=fde.PRECOND_MGM, tol=1e-8, restart=20, max_outer=100, omega=0.7,
                       cycles=1, coarse=fde.COARSE_SWEEPS, coarse_sweeps=3)
for name, m in (("slab x1", fde.SlabMarch(p, p.n, p.n, 8, cfg, rank=0, world=1)),
                ("single", fde.March(p, p.n, p.n, 8, cfg))):
    for _ in range(2):
        m.step()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            m.step()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
    span = ks[-1][1] - ks[0][0]
    print(f"== {name}: {steps} steps, span {span / 1e3 / steps:.2f} ms/step, {len(ks) // steps} device activities/step")
    fam = defaultdict(lambda: [0, 0.0])
    for a, b, nm in ks:
        k = nm.replace("(anonymous namespace)::", "").replace("fde_b200::", "").replace("void ", "").split("(")[0][:60]
        fam[k][0] += 1
        fam[k][1] += b - a
    for k, (c, t) in sorted(fam.items(), key=lambda kv: -kv[1][1])[:22]:
        print(f"  {t / 1e3 / steps:7.3f} ms/step {c // steps:5d} x {t / c:7.2f} us  {k}")
    del m
