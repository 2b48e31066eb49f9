"""BASELINE cfg5: operator-apply and V-cycle microbenchmark sweep on one GPU.

For n in {511, 1023, 2047, 4095, 8191}: one CN-WSGD operator apply and one
zero-guess V-cycle (omega 0.7, 3 coarsest sweeps) of the cfg5 operator
(reference coefficient preset 1, alpha 1.7, beta 1.3, tau 1/64) on seeded
U[-1, 1] vectors, timed with CUDA events after an L2 flush (median of 10),
reported as algorithmic GB/s and fraction of the measured HBM peak
(apply 48 N bytes; V-cycle sum over levels of
168 N_l + 16 N_{l+1}, 152 N_last on the coarsest).

    python tools/cfg5_sweep.py [out.json]
"""
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_1706_06844_b200 as fde

peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
hbm = float(peaks.get("hbm_gbs", 6551.7))
dev = torch.device("cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=dev)


def timed(fn, reps=10):
    out = []
    for r in range(reps + 2):
        flush.fill_(float(r))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if r >= 2:
            out.append(a.elapsed_time(b) / 1e3)
    return statistics.median(out)


rows = []
for n in (511, 1023, 2047, 4095, 8191):
    p = fde.Problem.preset_config(5, steps=1)
    op = fde.StructuredFdeOperator.assemble(p, n, n, 1, 1)
    g = torch.Generator(device=dev).manual_seed(n)
    x = torch.rand(n * n, dtype=torch.float64, device=dev, generator=g) * 2 - 1
    y = torch.empty_like(x)
    t_apply = timed(lambda: op.apply(x, y))
    h = fde.MgHierarchy.build_geometric(p, n, n, 1, 1, 0.7, fde.COARSE_SWEEPS, 3)
    dims = h.dims()
    z = torch.zeros_like(x)
    t_v = timed(lambda: h.vcycle(x, z, zero_guess=True))
    N = [a * b for a, b in dims]
    b_v = sum(168 * N[l] + 16 * N[l + 1] for l in range(len(N) - 1)) + 152 * N[-1]
    b_a = 48 * n * n
    row = {"n": n, "unknowns": n * n, "levels": len(dims),
           "apply_us": t_apply * 1e6, "apply_GBps": b_a / t_apply / 1e9,
           "apply_frac_hbm": b_a / t_apply / 1e9 / hbm,
           "vcycle_us": t_v * 1e6, "vcycle_GBps": b_v / t_v / 1e9,
           "vcycle_frac_hbm": b_v / t_v / 1e9 / hbm}
    rows.append(row)
    print(json.dumps(row), flush=True)
    del op, h, x, y, z
    torch.cuda.empty_cache()

out = {"config": "cfg5 sweep: apply + zero-guess V-cycle, L2 flushed, median of 10, one B200",
       "hbm_peak_GBps": hbm, "rows": rows}
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(json.dumps(out, indent=1))
