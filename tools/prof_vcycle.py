"""V-cycle timing (CUDA events, L2 warm) for cfg4 / cfg2 / cfg1 hierarchies:
python tools/prof_vcycle.py [cfg ...]; toggle the fused coarse tail with
FDE_MG_TAIL=0/1 and PDL with FDE_PDL=0/1."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1706_06844_b200 as fde

for cfg in [int(a) for a in sys.argv[1:]] or [4, 2, 1]:
    p = fde.Problem.preset_config(cfg)
    n = p.n
    h = fde.MgHierarchy.build_geometric(p, n, n, p.steps, 1, 0.7, fde.COARSE_SWEEPS, 3)
    b = torch.rand(n * n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    for _ in range(5):
        h.vcycle(b, x, zero_guess=True)
    torch.cuda.synchronize()
    # replay a captured V-cycle: device time without host launch overhead
    g = torch.cuda.CUDAGraph()
    k0 = fde.kernel_launches()
    with torch.cuda.graph(g):
        h.vcycle(b, x, zero_guess=True)
    launches = fde.kernel_launches() - k0
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    e.synchronize()
    print(f"cfg{cfg} n={n} levels={h.depth()} tail={os.environ.get('FDE_MG_TAIL', '1')} "
          f"pdl={os.environ.get('FDE_PDL', '1')}: V-cycle {s.elapsed_time(e) / reps * 1e3:.1f} us, "
          f"{launches} launches")
