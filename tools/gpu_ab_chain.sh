#!/bin/bash
# A/B of the Gram-Schmidt chain across build/var_*: per-launch durations under ncu (two GMRES
# steps' chains of cfg4), L2 read sectors of one chain, and bench steps/s of cfg4 / cfg1 / cfg2.
for d in main build/var_*; do
  [ -e "$d" ] || [ "$d" = main ] || continue
  if [ "$d" = main ]; then unset FDE_B200_LIB; else export FDE_B200_LIB=$d/libfde_b200.so; fi
  echo "== $d"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mgs_chain --csv python tools/prof_step.py 4 2 2>/dev/null | grep gpu__time | awk -F\",\" '{print $NF}' | tr -d \" | head -12 | tr "\n" " "; echo
  ncu --metrics lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:k_mgs_chain -s 8 -c 1 --csv python tools/prof_step.py 4 2 2>/dev/null | grep lts__ | awk -F\",\" '{print "sectors", $NF}'
  for rep in 1 2; do
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-traffic 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['configs']
print('   cfg4 %.2f' % d['value'], 'cfg1 %.1f cfg2 %.1f' % (c['cfg1']['steps_per_s'], c['cfg2']['steps_per_s']), ' '.join('%s %.1f' % (k[5:], v['steps_per_s']) for k, v in c.items() if k.startswith('cfg3_gm')))"
  done
done
