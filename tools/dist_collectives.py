"""Collectives per cfg4 time step of the y-slab march (counted by the C++
transport) on P virtual ranks of one GPU, with the slab-level plan.
usage: python tools/dist_collectives.py [n] [P ...]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1706_06844_b200 as fde

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2047
ranks = [int(v) for v in sys.argv[2:]] or [2, 4, 8]
cfg = fde.DriverConfig(precond=fde.PRECOND_MGM, tol=1e-8, restart=20, max_outer=100, omega=0.7,
                       cycles=1, coarse=fde.COARSE_SWEEPS, coarse_sweeps=3)
p = fde.Problem.preset_config(4, steps=8)
rows = []
for P in ranks:
    u, its, res, nc1 = fde.vdist_run(p, n, n, 8, cfg, P, "march", nrun=1)
    u, its2, res, nc2 = fde.vdist_run(p, n, n, 8, cfg, P, "march", nrun=2)
    rows.append({"n": n, "ranks": P, "iterations_step2": its2[1], "collectives_step2": nc2 - nc1,
                 "collectives_per_iteration": (nc2 - nc1) / max(its2[1], 1)})
    print(json.dumps(rows[-1]), flush=True)
