"""Kernel timeline of cfg4 (or argv[2]) time steps (CUPTI via torch.profiler): total span,
sum of kernel durations, gaps, and the per-kernel-family totals."""
import sys
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1706_06844_b200 as fde

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg_id = int(sys.argv[2]) if len(sys.argv) > 2 else 4  # BASELINE config (3: GMRES(30))
p = fde.Problem.preset_config(cfg_id, steps=8)
cfg = fde.DriverConfig(precond=fde.PRECOND_MGM, tol=1e-8, restart=30 if cfg_id == 3 else 20, max_outer=100, omega=0.7,
                       cycles=1, coarse=fde.COARSE_SWEEPS, coarse_sweeps=3)
m = fde.March(p, p.n, p.n, 8, cfg)
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
busy = sum(b - a for a, b, _ in ks)
gaps = [ks[i + 1][0] - ks[i][1] for i in range(len(ks) - 1)]
print(f"{steps} steps: span {span / 1e3:.2f} ms, kernels {len(ks)}, busy {busy / 1e3:.2f} ms, "
      f"gaps {sum(g for g in gaps if g > 0) / 1e3:.2f} ms (median gap {sorted(gaps)[len(gaps) // 2]:.2f} us)")
fam = defaultdict(lambda: [0, 0.0])
for a, b, nm in ks:
    k = nm.replace("(anonymous namespace)::", "").replace("fde_b200::", "").replace("void ", "").split("(")[0][:50]
    fam[k][0] += 1
    fam[k][1] += b - a
for k, (c, t) in sorted(fam.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {t / 1e3 / steps:7.3f} ms/step {c // steps:5d} x {t / c:7.2f} us  {k}")
# coarse-tail segments: maximal runs of short kernels (< 12 us), span incl. gaps
runs, cur = [], None
for a, b, nm in ks:
    if b - a < 12.0:
        cur = [a, b, 1] if cur is None else [cur[0], b, cur[2] + 1]
    else:
        if cur is not None and cur[2] >= 3:
            runs.append(cur)
        cur = None
if cur is not None and cur[2] >= 3:
    runs.append(cur)
tail = sum(b - a for a, b, _ in runs)
print(f"short-kernel runs (>=3 consecutive kernels < 12 us): {len(runs) // steps}/step, "
      f"{tail / 1e3 / steps:.3f} ms/step span, {sum(c for *_, c in runs) // steps} kernels/step")
big = [g for g in gaps if g > 5.0]
print(f"gaps > 5 us: {len(big) // steps}/step, {sum(big) / 1e3 / steps:.3f} ms/step; "
      f"gaps <= 5 us: {sum(g for g in gaps if 0 < g <= 5.0) / 1e3 / steps:.3f} ms/step")
small = [b - a for a, b, _ in ks if b - a < 12.0]
print(f"kernels < 12 us: {len(small) // steps}/step, {sum(small) / 1e3 / steps:.3f} ms/step busy")
# the largest gaps with their neighbours
order = sorted(range(len(gaps)), key=lambda i: -gaps[i])[:12]
for i in sorted(order):
    nm = lambda s: s.replace("(anonymous namespace)::", "").replace("fde_b200::", "").split("(")[0][-38:]
    print(f"  gap {gaps[i]:8.1f} us after {nm(ks[i][2]):38s} before {nm(ks[i + 1][2])}")
