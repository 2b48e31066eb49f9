#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the dev container (where /root/reference exists and oracle/_ref is
built):  python tools/make_golden.py [--long]
--long adds the full-size cfg3 / cfg4 trajectories (minutes of CPU each).

Full-size vectors are summarised, not stored: per step the l2 norm, three
weighted checksums with counter-hash weights (golden_weights below, also used
by the tests) and, for the final step, 2048 sampled entries.
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
from oracles import oracle, reflib, spec  # noqa: E402
from golden_util import summarize, sample_idx  # noqa: E402

OUT = ROOT / "tests" / "golden"


def save(name, **arrs):
    np.savez_compressed(OUT / f"{name}.npz", **arrs)
    print("wrote", name, {k: getattr(v, "shape", None) for k, v in arrs.items()}, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--long", action="store_true")
    ap.add_argument("--only", default="")
    ap.add_argument("--oracle-bicgstab", action="store_true",
                    help="cfg3 BiCGSTAB trajectories from the C oracle (no reference code exists)")
    args = ap.parse_args()
    R = reflib()
    assert R is not None, "build oracle/_ref first (make -C oracle ref)"
    OUT.mkdir(parents=True, exist_ok=True)
    only = set(args.only.split(",")) if args.only else None

    def want(n):
        return only is None or n in only

    if want("weights"):
        d = {}
        for gamma in (1.1, 1.3, 1.5, 1.6, 1.7, 1.8, 1.9, 2.0):
            for pq in (0, 1):
                g, w = R.weights(gamma, 64, pq)
                d[f"g_{gamma}_{pq}"], d[f"w_{gamma}_{pq}"] = g, w
        save("weights", **d)

    if want("toeplitz"):
        d = {}
        rng = np.random.default_rng(11)
        for n in (1, 2, 3, 7, 8, 31, 33, 64, 100):
            x = rng.uniform(-1, 1, n)
            for gamma, pq in ((1.5, 0), (1.8, 0), (1.1, 1)):
                y, yt = R.toeplitz_both(gamma, x, pq)
                d[f"x_{n}"] = x
                d[f"y_{n}_{gamma}_{pq}"], d[f"yt_{n}_{gamma}_{pq}"] = y, yt
        save("toeplitz", **d)

    if want("plans"):
        d = {}
        for cfg in (1, 2, 3, 4, 5):
            dims, r0 = R.plan(spec(cfg))
            d[f"plan_{cfg}"] = np.array(dims)
            d[f"ratio0_{cfg}"] = np.array(r0)
        for n in (511, 1023, 4095, 8191):
            dims, r0 = R.plan(spec(5, n1=n, n2=n))
            d[f"plan_5_{n}"] = np.array(dims)
        save("plans", **d)

    if want("apply"):  # operator / rhs / diagonal / V-cycle on small grids
        d = {}
        rng = np.random.default_rng(7)
        for cfg, n1, n2 in ((1, 63, 63), (2, 31, 47), (3, 64, 33), (4, 47, 31), (5, 63, 63)):
            s = spec(cfg, n1=n1, n2=n2, steps=4)
            x = rng.uniform(-1, 1, n1 * n2)
            d[f"x_{cfg}"] = x
            d[f"y_{cfg}"] = R.apply(s, x, 1)
            d[f"yr_{cfg}"] = R.apply(s, x, -1)
            d[f"diag_{cfg}"] = R.diagonal(s)
            for coarse in (0, 1, 2):
                sc = spec(cfg, n1=n1, n2=n2, steps=4, coarse=coarse)
                d[f"v_{cfg}_{coarse}"] = R.vcycle(sc, x)
            d[f"p2_{cfg}"] = R.vcycle(spec(cfg, n1=n1, n2=n2, steps=4, precond=1), x)
        save("apply", **d)

    if want("cfg1"):
        s = spec(1)
        r = R.march(s, record=True)
        us = r["u_steps"]
        save("cfg1", its=r["its"], res=r["res"], u_final=r["u"],
             u_step1=us[0], u_step32=us[31], **summarize(us))
        s2 = spec(1, precond=1)
        r2 = R.march(s2, record=True)
        save("cfg1_p2", its=r2["its"], res=r2["res"], u_final=r2["u"], **summarize(r2["u_steps"]))

    if want("cfg2"):
        s = spec(2, steps=4)
        r = R.march(s, record=True)
        save("cfg2_4steps", its=r["its"], res=r["res"], **summarize(r["u_steps"]),
             samples=r["u"][sample_idx(255 * 255)])

    if args.oracle_bicgstab:
        O = oracle()
        for name, coarse in (("cfg3_bicgstab_sweeps", 1), ("cfg3_bicgstab_lu", 0)):
            if not want(name):
                continue
            t0 = time.time()
            r = O.march(spec(3, coarse=coarse), record=True, solver=1)
            save(name, its=r["its"], res=r["res"], **summarize(r["u_steps"]),
                 samples=r["u"][sample_idx(r["u"].size)], seconds=np.array(time.time() - t0),
                 source=np.array("oracle/fde_oracle.c bicgstab (not in the reference)"))

    if args.long:
        for name, s in (("cfg3_lu", spec(3, coarse=0)), ("cfg3_sweeps", spec(3, coarse=1)),
                        ("cfg4", spec(4))):
            if not want(name):
                continue
            t0 = time.time()
            r = R.march(s, record=True)
            n = r["u"].size
            save(name, its=r["its"], res=r["res"], **summarize(r["u_steps"]),
                 samples=r["u"][sample_idx(n)], seconds=np.array(time.time() - t0))


if __name__ == "__main__":
    main()
