"""SASS window of an ncu report with stall samples: python tools/ncu_window.py rep kernel_substr addr_suffix [before after]"""
import csv, io, subprocess, sys
rep, pat, addr = sys.argv[1:4]
before = int(sys.argv[4]) if len(sys.argv) > 4 else 30
after = int(sys.argv[5]) if len(sys.argv) > 5 else 5
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
for b in txt.split('"Kernel Name",')[1:]:
    name, rest = b.split("\n", 1)
    if pat not in name:
        continue
    rows = list(csv.DictReader(io.StringIO(rest)))
    stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    for i, r in enumerate(rows):
        if r["Address"].endswith(addr):
            for j in range(max(0, i - before), min(len(rows), i + after + 1)):
                q = rows[j]
                top = sorted(((int(q[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
                print(f"{q['Address'][-5:]} {q['Warp Stall Sampling (All Samples)']:>5s} {q['Instructions Executed']:>8s} {q['Source'].strip()[:70]:70s} " + ", ".join(f"{k}={v}" for v, k in top if v))
    break
