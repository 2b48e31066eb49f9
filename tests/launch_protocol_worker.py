"""Worker of test_gpu_launch_protocol.py: SHA-256 of many operator applies and V-cycles at
ragged sizes (run once with FDE_PDL=1 and once with FDE_PDL=0; the digests must be equal)."""
import hashlib
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1706_06844_b200 as fde

fde.load_library()
h = hashlib.sha256()
rng = np.random.default_rng(7)
# sizes that exercise every line-kernel family and both transposed / gathered column input
for cfg, n1, n2 in [(4, 2047, 2047), (4, 1023, 2047), (3, 1023, 1023), (2, 511, 1023), (2, 255, 255),
                    (1, 127, 63), (4, 4095, 130)]:
    p = fde.Problem.preset_config(cfg, steps=8)
    op = fde.StructuredFdeOperator.assemble(p, n1, n2, 8, 1)
    x = torch.tensor(rng.uniform(-1, 1, n1 * n2), device="cuda")
    y = torch.empty_like(x)
    reps = 60 if n1 * n2 > 10**6 else 200
    for r in range(reps):
        op.apply(x, y)
        x, y = y, x  # feed the result back: every launch depends on the one before
        if r % 20 == 19:
            x = x / x.abs().max()
    h.update(x.cpu().numpy().tobytes())
for cfg in (4, 2, 1):
    p = fde.Problem.preset_config(cfg)
    n = p.n
    mg = fde.MgHierarchy.build_geometric(p, n, n, p.steps, 1, 0.7, fde.COARSE_SWEEPS, 3)
    b = torch.tensor(rng.uniform(-1, 1, n * n), device="cuda")
    x = torch.empty_like(b)
    for r in range(30 if cfg == 4 else 150):
        mg.vcycle(b, x, zero_guess=True)
        b = x / x.abs().max()
    h.update(b.cpu().numpy().tobytes())
# whole time steps (GMRES + V-cycle + the one-launch Gram-Schmidt): iteration counts and solutions
for cfg, steps in ((2, 8), (4, 3)):
    p = fde.Problem.preset_config(cfg, steps=steps)
    dc = fde.DriverConfig(precond=fde.PRECOND_MGM, tol=1e-8, restart=20, max_outer=100, omega=0.7,
                          cycles=1, coarse=fde.COARSE_SWEEPS, coarse_sweeps=3)
    m = fde.March(p, p.n, p.n, steps, dc)
    for _ in range(steps):
        it, res = m.step()
        h.update(str(it).encode())
    h.update(m.solution().tobytes())
print("DIGEST", h.hexdigest())
