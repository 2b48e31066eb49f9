"""Per-CUDA-source-line warp-stall samples from an ncu report (cuda,sass view).
usage: python tools/ncu_lines.py REP KERNEL_SUBSTR [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur_file, cur_fn, hdr = None, None, None
agg = {}
tot = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        cur_fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        stall = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if pat not in (cur_fn or "") or hdr is None or r[0] == "":
        continue
    if not r[si].isdigit():
        continue
    s = int(r[si])
    if s == 0:
        continue
    key = (cur_file, int(r[0]))
    d = {"src": r[1].strip()[:70], "n": s}
    for i, h in stall:
        d[h] = int(r[i]) if r[i].isdigit() else 0
    agg[key] = d
    tot += s
print(f"{tot} samples in {pat}")
for (f, ln), d in sorted(agg.items(), key=lambda kv: -kv[1]["n"])[:top]:
    st = sorted(((v, k) for k, v in d.items() if k not in ("src", "n")), reverse=True)[:3]
    print(f"{d['n']:6d} {100 * d['n'] / tot:5.1f}% {f}:{ln:<5d} {d['src']:70s} " + ", ".join(f"{k}={v}" for v, k in st if v))
