#!/bin/bash
# One GPU iteration: parity subset, apply timing, per-kernel launch times.
# usage (on the box): bash tools/gpu_iter.sh [pytest -k expr] [n]
K=${1:-"apply"}
N=${2:-2047}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "$K" > gpurun_out/iter_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/iter_pytest.log
tail -3 gpurun_out/iter_pytest.log
timeout 120 python tools/prof_apply.py $N 8 > gpurun_out/iter_apply.log 2>&1
cat gpurun_out/iter_apply.log
timeout 300 ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:line_kernel -s 6 -c 6 --csv python tools/prof_apply.py $N 8 > gpurun_out/iter_ncu.csv 2>/dev/null
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/iter_ncu.csv")) if len(r)>10]
h=rows[0]
ki,mi,vi,ii=h.index("Kernel Name"),h.index("Metric Name"),h.index("Metric Value"),h.index("ID")
for r in rows[1:]:
    print(r[ii], r[ki][:60], r[mi], r[vi])
PY
