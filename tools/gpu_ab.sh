#!/bin/bash
# A/B of build/var_* against the main build on one box: apply check + warm
# apply time (tools/var_bench.py), then cfg4 steps/s (bench.py --steps-only), twice.
mkdir -p gpurun_out
SIZES=${SIZES:-2047}
for rep in 1 2; do
for d in main build/var_*; do
  if [ "$d" = main ]; then unset FDE_B200_LIB; else export FDE_B200_LIB=$d/libfde_b200.so; fi
  python tools/var_bench.py $SIZES 2>&1 | grep "^\[" | cut -c1-200
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --steps-only 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   steps/s %.2f  ms/step %.3f' % (d['value'], d['ms_per_step']))"
done
done
