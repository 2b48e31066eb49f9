#!/bin/bash
# A/B of build/var_* against the main build: graph-replayed V-cycles (cfg4, cfg2) and cfg4 steps/s, twice.
mkdir -p gpurun_out
for rep in 1 2; do
for d in main build/var_*; do
  if [ "$d" = main ]; then unset FDE_B200_LIB; else export FDE_B200_LIB=$d/libfde_b200.so; fi
  echo "[$d]"
  python tools/prof_vcycle.py 4 2 2>&1 | grep V-cycle | cut -c1-80
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --steps-only 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   steps/s %.2f  ms/step %.3f' % (d['value'], d['ms_per_step']))"
done
done
