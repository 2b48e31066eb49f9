for rep in 1 2; do
for d in main build/var_*; do
  [ -e "$d" ] || [ "$d" = main ] || continue
  if [ "$d" = main ]; then unset FDE_B200_LIB; else export FDE_B200_LIB=$d/libfde_b200.so; fi
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-traffic 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['configs']
print('$d', 'cfg4 %.2f' % d['value'], 'cfg1 %.1f cfg2 %.1f' % (c['cfg1']['steps_per_s'], c['cfg2']['steps_per_s']), ' '.join('%s %.1f' % (k[5:], v['steps_per_s']) for k, v in c.items() if k.startswith('cfg3_gm')))"
done
done
