"""Variant check + timing of the operator apply (for kernel experiments).
usage: FDE_B200_LIB=... python tools/var_bench.py [n ...]
Prints the relative error vs the CPU oracle (n <= 2047) and per-kernel device
times (torch profiler / CUPTI) of the line kernels over 10 applies."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_1706_06844_b200 as fde
from oracles import oracle, spec

sizes = [tuple(int(v) for v in a.split("x")) if "x" in a else (int(a), int(a)) for a in sys.argv[1:]] or [(2047, 2047)]
orc = oracle()
tag = os.environ.get("FDE_B200_LIB", "main")
for n1, n2 in sizes:
    n = f"{n1}x{n2}"
    p = fde.Problem.preset_config(4, steps=8)
    op = fde.StructuredFdeOperator.assemble(p, n1, n2, 8, 1)
    x = np.random.default_rng(n1 + n2).uniform(-1, 1, n1 * n2)
    xd = torch.tensor(x, device="cuda")
    y = op.apply(xd).cpu().numpy()
    yo = orc.apply(spec(4, n1=n1, n2=n2, steps=8), x)
    err = np.linalg.norm(y - yo) / np.linalg.norm(yo)
    yd = torch.empty_like(xd)
    for _ in range(3):
        op.apply(xd, yd)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        op.apply(xd, yd)
    e.record()
    e.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            op.apply(xd, yd)
        torch.cuda.synchronize()
    ks = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            k = ev.name.replace("(anonymous namespace)::", "").replace("fde_b200::", "")
            k = k.replace("void ", "").split("(")[0].replace("fft_line_kernel", "L").replace("Pass", "")[:40]
            ks.setdefault(k, []).append(ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total)
    print(f"[{Path(tag).parent.name or tag}] n={n} err={err:.2e} apply(L2 warm)={s.elapsed_time(e) / 20 * 1e3:.1f} us  " +
          "  ".join(f"{k}={np.median(v):.1f}" for k, v in sorted(ks.items())))
