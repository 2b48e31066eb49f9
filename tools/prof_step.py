"""Profiling driver: N CN-WSGD steps of a BASELINE config (default cfg4)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1706_06844_b200 as fde

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = fde.Problem.preset_config(cfg_id, steps=max(steps, 1))
n = p.n
cfg = fde.DriverConfig(precond=fde.PRECOND_MGM, tol=1e-8, restart=20, max_outer=100, omega=0.7,
                       cycles=1, coarse=fde.COARSE_SWEEPS, coarse_sweeps=3)
m = fde.March(p, n, n, steps, cfg)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for k in range(steps):
    l0 = fde.kernel_launches()
    s.record()
    it, res = m.step()
    e.record()
    e.synchronize()
    print(f"step {k + 1}: {it} its, {s.elapsed_time(e):.2f} ms, {fde.kernel_launches() - l0} launches")
