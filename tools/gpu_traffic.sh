#!/bin/bash
# DRAM traffic per apply (every kernel, write-backs included) and warm / flushed apply time, main build and build/var_*
mkdir -p gpurun_out
for d in main build/var_*; do
  [ -e "$d" ] || [ "$d" = main ] || continue
  if [ "$d" = main ]; then unset FDE_B200_LIB; else export FDE_B200_LIB=$d/libfde_b200.so; fi
  echo "== $d"
  python tools/var_bench.py 2047 1023x2047 2>&1 | grep "^\[" | cut -c1-70
  python tools/prof_apply.py 2047 6 2>&1 | tail -2
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
    -k regex:"line_kernel|transpose|elementwise" --csv --log-file /tmp/traffic.csv python tools/traffic_probe.py 2047 3 > /dev/null 2>&1
  python tools/traffic_probe.py --parse /tmp/traffic.csv
done
