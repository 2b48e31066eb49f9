"""Summarise `ncu --page source --csv --print-source sass` output: warp-stall
samples per opcode and the hottest instructions, per kernel."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = txt.split('"Kernel Name",')[1:]
for b in blocks:
    name, rest = b.split("\n", 1)
    if pat and pat not in name:
        continue
    rows = list(csv.DictReader(io.StringIO(rest)))
    stall_cols = [c for c in rows[0] if c.startswith("stall_")]
    tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    print(f"== {name.strip()} : {len(rows)} SASS lines, {tot} samples")
    by_op = defaultdict(lambda: defaultdict(int))
    inst_by_op = defaultdict(int)
    for r in rows:
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        op = op.split(".")[0]
        inst_by_op[op] += int(r["Instructions Executed"] or 0)
        by_op[op]["samples"] += int(r["Warp Stall Sampling (All Samples)"] or 0)
        for c in stall_cols:
            by_op[op][c] += int(r[c] or 0)
    print(f"{'op':10s} {'warp-inst':>10s} {'samples':>8s}  top stalls")
    for op, d in sorted(by_op.items(), key=lambda kv: -kv[1]["samples"])[:18]:
        top = sorted(((d[c], c[6:]) for c in stall_cols), reverse=True)[:4]
        print(f"{op:10s} {inst_by_op[op]:10d} {d['samples']:8d}  " +
              ", ".join(f"{k}={v}" for v, k in top if v))
    agg = defaultdict(int)
    for r in rows:
        for c in stall_cols:
            agg[c] += int(r[c] or 0)
    print("all:", ", ".join(f"{c[6:]}={v}" for c, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))
    print("hottest:")
    for r in sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:int(sys.argv[3]) if len(sys.argv) > 3 else 15]:
        top = sorted(((int(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        print(f"  {r['Address'][-5:]} {r['Warp Stall Sampling (All Samples)']:>6s} {r['Source'].strip()[:60]:60s} " +
              ", ".join(f"{k}={v}" for v, k in top if v))
