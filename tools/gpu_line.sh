#!/bin/bash
# Line-kernel iteration on the GPU box: warm timing of the apply at the cfg4 /
# cfg5 sizes, then one `ncu --set full` capture of the kernels of one n = 2047
# apply (transpose, column pass, row pass).  usage: bash tools/gpu_line.sh [tag]
TAG=${1:-cur}
mkdir -p gpurun_out
python tools/var_bench.py 2047 1023x2047 2>&1 | grep "^\[" | tee gpurun_out/var_$TAG.txt
python tools/prof_apply.py 2047 4 > gpurun_out/plain_$TAG.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"line_kernel|transpose" -s 6 -c 3 \
  -f -o gpurun_out/apply_$TAG python tools/prof_apply.py 2047 4 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
