"""Small hot-path run for compute-sanitizer (tools/sanitize.sh): cfg1 time
step, cfg2 apply + V-cycle, and one apply + V-cycle at n = 1023 and one apply
at n = 2047 so the paired line kernels (bulk copies, mbarriers, tensor-memory
stash, padded exchange slots) are covered."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1706_06844_b200 as fde

cfg = fde.DriverConfig(precond=fde.PRECOND_MGM, tol=1e-8, restart=20, max_outer=100, omega=0.7,
                       cycles=1, coarse=fde.COARSE_SWEEPS, coarse_sweeps=3)
p1 = fde.Problem.preset_config(1, seed=0)
m = fde.March(p1, 63, 63, 64, cfg)
print("cfg1 step:", m.step()[0], "iterations")
for c, n in ((2, 255), (4, 1023)):
    p = fde.Problem.preset_config(c, steps=8)
    op = fde.StructuredFdeOperator.assemble(p, n, n, 8, 1)
    x = torch.tensor(np.random.default_rng(n).uniform(-1, 1, n * n), device="cuda")
    y = op.apply(x)
    h = fde.MgHierarchy.build_geometric(p, n, n, 8, 1, 0.7, fde.COARSE_SWEEPS, 3)
    z = h.vcycle(x)
    print(f"n={n}: |Ax|={float(y.norm()):.6e} |Vx|={float(z.norm()):.6e}")
if len(sys.argv) > 1 and sys.argv[1] == "big":
    p = fde.Problem.preset_config(4, steps=8)
    op = fde.StructuredFdeOperator.assemble(p, 2047, 2047, 8, 1)
    x = torch.rand(2047 * 2047, dtype=torch.float64, device="cuda")
    print("n=2047:", float(op.apply(x).norm()))
torch.cuda.synchronize()
print("done")
