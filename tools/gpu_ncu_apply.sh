#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:line_kernel -s 4 -c 2 -o gpurun_out/apply_full2 python tools/prof_apply.py 2047 4 > gpurun_out/ncu_full2.log 2>&1; echo "ncu rc=$?"
timeout 300 python tools/var_bench.py 2047 1023x2047 2>&1 | grep "^\["
