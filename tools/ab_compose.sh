cd $GRAFT_REPO_ROOT
for comp in triples pairs singles none; do
  for c in 2 3; do
    [ "$c" = 3 ] && [ "$comp" = none ] && continue
    timeout 300 python bench.py --config $c --compose $comp --steps 10 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$comp', 'c$c', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['ms_per_launch'],3), round(d['config']['mean_rows_per_iteration'],2), d['clocks']['sm_mhz'])"
  done
done
