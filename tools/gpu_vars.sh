#!/bin/bash
# A/B of build/var_* against the main build: warm apply time, then per-kernel
# device time and L1 hit rate from a metrics-only ncu pass.
mkdir -p gpurun_out
SIZES=${SIZES:-2047}
for d in main build/var_*; do
  if [ "$d" = main ]; then unset FDE_B200_LIB; else export FDE_B200_LIB=$d/libfde_b200.so; fi
  python tools/var_bench.py $SIZES 2>&1 | grep "^\[" | cut -c1-60
  python tools/prof_apply.py 2047 4 > /dev/null 2>&1 &&
  ncu --metrics gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio \
    --clock-control none -k regex:"line_kernel" -s 4 -c 2 --csv python tools/prof_apply.py 2047 4 2>/dev/null | grep -E "paired" | awk -F'","' '{print "   ", substr($5,1,50), $(NF-2), $(NF)}' | tr -d '"'
done
