#!/bin/bash
# A/B of build/var_* (tools/build_variant.sh) against the main build on one box, two passes:
# apply check + warm apply time (tools/var_bench.py, SIZES), graph-replayed V-cycles when
# VCYCLE is set (tools/prof_vcycle.py, e.g. VCYCLE="4 2"), and cfg4 steps/s (bench.py --steps-only).
mkdir -p gpurun_out
SIZES=${SIZES:-2047}
for rep in 1 2; do
for d in main build/var_*; do
  [ -e "$d" ] || [ "$d" = main ] || continue
  if [ "$d" = main ]; then unset FDE_B200_LIB; else export FDE_B200_LIB=$d/libfde_b200.so; fi
  python tools/var_bench.py $SIZES 2>&1 | grep "^\[" | cut -c1-200
  [ -n "$VCYCLE" ] && python tools/prof_vcycle.py $VCYCLE 2>&1 | grep V-cycle | cut -c1-80
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --steps-only 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   steps/s %.2f  ms/step %.3f' % (d['value'], d['ms_per_step']))"
done
done
