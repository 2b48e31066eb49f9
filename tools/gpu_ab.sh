#!/bin/bash
# A/B of the main build against build/var_*: cfg4 bench steps/s (no CPU leg), alternating
mkdir -p gpurun_out
for rep in 1 2; do
  for d in main build/var_*; do
    if [ "$d" = main ]; then unset FDE_B200_LIB; else export FDE_B200_LIB=$d/libfde_b200.so; fi
    timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$d', round(d['value'],2), round(d['e2e']['value'],2), round(d['operator_apply']['seconds']*1e6,1))"
  done
done
unset FDE_B200_LIB
