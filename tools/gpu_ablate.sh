#!/bin/bash
# Timing-only ablation builds (build/var_*; results wrong by construction): per-kernel device
# time of one n = 2047 apply with programmatic launches off (FDE_PDL=0: no overlap between kernels).
mkdir -p gpurun_out
export FDE_PDL=0
for d in main build/var_*; do
  [ -e "$d" ] || [ "$d" = main ] || continue
  if [ "$d" = main ]; then unset FDE_B200_LIB; else export FDE_B200_LIB=$d/libfde_b200.so; fi
  python tools/var_bench.py 2047 2>&1 | grep "^\[" | cut -c1-200
done
