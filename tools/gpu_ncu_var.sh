#!/bin/bash
# ncu --set full capture of one n = 2047 apply for a variant build: bash tools/gpu_ncu_var.sh NAME TAG
NAME=$1; TAG=${2:-$1}
mkdir -p gpurun_out
if [ "$NAME" != main ]; then export FDE_B200_LIB=build/var_$NAME/libfde_b200.so; fi
python tools/prof_apply.py 2047 4 > gpurun_out/plain_$TAG.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"line_kernel|transpose" -s 6 -c 3 \
  -f -o gpurun_out/apply_$TAG python tools/prof_apply.py 2047 4 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu $NAME rc=$?"
