"""Long-scoreboard stall sites of each kernel in an ncu report (source page):
the top instructions by long_sb samples and the load each one waits behind.

    python tools/ncu_lsb_sites.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
seen = set()
for b in txt.split('"Kernel Name",')[1:]:
    name, rest = b.split("\n", 1)
    if name in seen:
        continue
    seen.add(name)
    rows = list(csv.DictReader(io.StringIO(rest)))
    tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    lsb = sum(int(r["stall_long_sb"] or 0) for r in rows)
    print(f"== {name.strip()}: {tot} samples, long_sb {lsb} ({100.0 * lsb / max(tot, 1):.1f} %)")
    idx = sorted(range(len(rows)), key=lambda i: -int(rows[i]["stall_long_sb"] or 0))[:top]
    for i in sorted(idx):
        r = rows[i]
        j = i - 1
        while j > 0 and not any(k in rows[j]["Source"] for k in ("LDG", "LDTM", "DEPBAR", "LDS", "LDL")):
            j -= 1
        print(f"  sass#{i:5d} long_sb={int(r['stall_long_sb']):4d} {r['Source'].strip()[:44]:44s}"
              f" waits on ({i - j:3d} back) {rows[j]['Source'].strip()[:52]}")
