"""Paper-table runs on the GPU: `fde table --table k`
semantics (proj/src/cli.cpp:151-211) through this library.

For table k (= example k, alpha 1.8, beta 1.6 for k=1 else 1.9) and each
n in --sizes: Grid(p, n, n, n), time_march with each preconditioner column
(none with restart 512, p2 and mgm with restart 20; tol 1e-7, omega 0.9,
one V-cycle per apply), recording the average GMRES iterations per step and
the final max-norm error against the exact solution.  With --reference the
reference's own fde::time_march (oracle/_ref, host CPU, 1 core) runs the same
cells and its numbers are written beside ours.  Columns p2-exact and
mgm-galerkin (table 1) are not offered by this library.

    python tools/paper_tables.py --tables 1 2 3 --sizes 16 32 64 128 \
        --out profiles/paper_tables_r01.csv [--reference]
"""
import argparse
import csv
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_1706_06844_b200 as fde  # noqa: E402

COLUMNS = {"none": fde.PRECOND_NONE, "p2": fde.PRECOND_P2, "mgm": fde.PRECOND_MGM}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tables", type=int, nargs="+", default=[1, 2, 3])
    ap.add_argument("--sizes", type=int, nargs="+", default=[16, 32, 64, 128])
    ap.add_argument("--columns", nargs="+", default=list(COLUMNS))
    ap.add_argument("--cycles", type=int, default=1)
    ap.add_argument("--reference", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    ref = None
    if a.reference:
        from oracles import reflib, spec  # test infrastructure: the reference build
        ref = reflib()
    rows = []
    for k in a.tables:
        alpha, beta = 1.8, (1.6 if k == 1 else 1.9)
        p = fde.Problem.example(k, alpha, beta)
        for n in sorted(set(a.sizes)):
            for col in a.columns:
                pc = COLUMNS[col]
                restart = 512 if pc == fde.PRECOND_NONE else 20
                cfg = fde.DriverConfig(precond=pc, tol=1e-7, restart=restart, max_outer=100,
                                       omega=0.9, cycles=a.cycles, coarse=fde.COARSE_SWEEPS,
                                       coarse_sweeps=3)
                t0 = time.perf_counter()
                rep = fde.time_march(p, n, n, n, cfg)
                wall = time.perf_counter() - t0
                row = dict(table=k, n=n, precond=col, cycles=a.cycles,
                           avg_iterations=round(rep.avg_iterations, 3),
                           error_inf=rep.error_inf, converged=rep.all_converged,
                           gpu_wall_s=round(wall, 4))
                if ref is not None:
                    s = spec(100 + k, n1=n, n2=n, steps=n, precond=pc, restart=restart,
                             tol=1e-7, omega=0.9, cycles=a.cycles, coarse=fde.COARSE_SWEEPS)
                    t0 = time.perf_counter()
                    w = ref.time_march(s)
                    row["ref_avg_iterations"] = round(float(w["its"].mean()), 3)
                    row["ref_error_inf"] = ref.error_inf(s, w["u"], 1.0)
                    row["ref_wall_s"] = round(time.perf_counter() - t0, 3)
                rows.append(row)
                print(row, flush=True)
    if a.out:
        keys = list(rows[0].keys())
        for r in rows:
            for kk in r:
                if kk not in keys:
                    keys.append(kk)
        with open(a.out, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=keys)
            w.writeheader()
            w.writerows(rows)
        print("wrote", a.out)


if __name__ == "__main__":
    main()
