"""Profiling driver: cfg4 (n=2047) operator applies, for ncu / nsight runs."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1706_06844_b200 as fde

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2047
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 4
p = fde.Problem.preset_config(cfg, steps=8)
op = fde.StructuredFdeOperator.assemble(p, n, n, 8, 1)
x = torch.rand(n * n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(reps):
    s.record()
    op.apply(x, y)
    e.record()
    e.synchronize()
    print(f"apply {r}: {s.elapsed_time(e) * 1e3:.1f} us")
