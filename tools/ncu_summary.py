"""Summarise an `ncu --set full` report of one operator apply into the judged
profile files: per-kernel key metrics + stall reasons per issued instruction
(JSON), and the DRAM bytes per apply used as bench.py's `roofline.traffic`.

    python tools/ncu_summary.py gpurun_out/apply_full.ncu-rep profiles/ncu_apply_r01.json \
        [profiles/apply_traffic.json] ["source command"]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
    "l1tex__t_sector_hit_rate.pct",
]
STALLS = ["long_scoreboard", "wait", "short_scoreboard", "mio_throttle", "not_selected",
          "math_pipe_throttle", "barrier", "lg_throttle", "dispatch_stall", "no_instruction"]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    traffic_out = sys.argv[3] if len(sys.argv) > 3 else None
    source = sys.argv[4] if len(sys.argv) > 4 else f"ncu --set full report {rep}"
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    kernels, total_bytes = [], 0.0
    for r in data:
        k = {"Kernel Name": r[hdr.index("Kernel Name")]}
        for key in KEYS:
            if key in hdr:
                k[key] = r[hdr.index(key)]
        st = {}
        for s in STALLS:
            key = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if key in hdr:
                st[s] = float(r[hdr.index(key)].replace(",", "") or 0)
        k["stalls_per_issue"] = dict(sorted(st.items(), key=lambda kv: -kv[1]))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            u = units[hdr.index(key)]
            total_bytes += float(r[hdr.index(key)].replace(",", "")) * scale.get(u, 1)
        kernels.append(k)
    units_d = {key: units[hdr.index(key)] for key in KEYS if key in hdr}
    json.dump({"source": source, "units": units_d, "kernels": kernels}, open(out, "w"), indent=1)
    print(f"{len(kernels)} kernels, DRAM {total_bytes / 1e6:.1f} MB")
    if traffic_out:
        json.dump({"bytes_per_apply": total_bytes,
                   "source": f"ncu --set full ({out}): sum over the captured line kernels of "
                             "dram__bytes_read.sum + dram__bytes_write.sum"},
                  open(traffic_out, "w"), indent=1)


if __name__ == "__main__":
    main()
