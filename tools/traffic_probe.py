"""DRAM traffic of one operator apply, every kernel counted.

Run under `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum` (bench.py
does this in a subprocess after its timed legs).  The launch sequence is

    flush, flush, [apply, flush] x REPS

where flush writes a 512 MB buffer (> L2), so every dirty line an apply leaves
in L2 (the Q scratch, the output) is written back inside the flush that
follows it.  bytes(apply) = bytes of the apply's kernels (transpose, column
pass, row pass) + bytes of the following flush - bytes of a flush alone.

    python tools/traffic_probe.py [n] [reps]          # the launch sequence
    python tools/traffic_probe.py --parse FILE.csv    # -> JSON on stdout
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def parse(path):
    rows = list(csv.reader(open(path, errors="replace")))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
    h = rows[hdr]
    ik, im, iv, iu, iid = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value",
                                                  "Metric Unit", "ID"))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    launches = {}
    for r in rows[hdr + 1:]:
        if len(r) <= iv or not r[iid].isdigit():
            continue
        d = launches.setdefault(int(r[iid]), {"name": r[ik], "bytes": 0.0, "rd": 0.0, "wr": 0.0})
        if r[im] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
            d["bytes"] += v
            d["rd" if "read" in r[im] else "wr"] += v
    seq = [launches[k] for k in sorted(launches)]
    is_apply = lambda d: ("line_kernel" in d["name"]) or ("transpose" in d["name"])
    # flush alone: a non-apply launch that follows another non-apply launch
    alone = [b["bytes"] for a, b in zip(seq, seq[1:]) if not is_apply(a) and not is_apply(b)]
    if not alone:
        raise ValueError("no standalone flush launch in the capture")
    base = alone[-1]
    per_apply, kernels, cur, names = [], [], 0.0, []
    for d in seq:
        if is_apply(d):
            cur += d["bytes"]
            names.append({"kernel": d["name"].split("(")[0].split("::")[-1][:48],
                          "read_MB": round(d["rd"] / 1e6, 1), "write_MB": round(d["wr"] / 1e6, 1)})
        elif names:
            per_apply.append(cur + d["bytes"] - base)
            names.append({"kernel": "write-back during the following flush",
                          "extra_MB": round((d["bytes"] - base) / 1e6, 1)})
            kernels, cur, names = names, 0.0, []
    if not per_apply:
        raise ValueError("no apply in the capture")
    per_apply.sort()
    return {"bytes_per_apply": per_apply[len(per_apply) // 2], "applies": len(per_apply),
            "flush_alone_bytes": base, "kernels_per_apply": kernels}


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--parse":
        print(json.dumps(parse(sys.argv[2])))
        return
    import torch
    sys.path.insert(0, str(ROOT))
    import paper_1706_06844_b200 as fde
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2047
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    p = fde.Problem.preset_config(4, steps=8)
    op = fde.StructuredFdeOperator.assemble(p, n, n, 8, 1)
    x = torch.rand(n * n, dtype=torch.float64, device="cuda") * 2 - 1
    y = torch.empty_like(x)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    flush.fill_(0.0)
    flush.fill_(1.0)
    for r in range(reps):
        op.apply(x, y)
        flush.fill_(float(r))
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
