"""Summarise an ncu launch list (gpu__time_duration.sum CSV): per-kernel totals
over the last `steps` of `total` equal steps."""
import collections
import csv
import re
import sys

path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5  # tail fraction of launches to keep
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi, gi, bi = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Grid Size", "Block Size"))
keep = rows[int(len(rows) * (1 - frac)):]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in keep:
    raw = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    raw = raw.replace("fde_b200::", "").replace("void ", "")
    name = re.sub(r"\(.*", "", raw)[:48]
    key = f"{name} g{r[gi]} b{r[bi]}"
    agg[key][0] += 1
    agg[key][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{path}: {len(keep)} launches, {tot / 1e6:.3f} ms (serialised)")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"  {t / 1e6:7.3f} ms {100 * t / tot:5.1f}% {c:5d} x {t / c / 1e3:7.2f} us  {k}")
