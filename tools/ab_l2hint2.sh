# A/B: L2 residency hint on the config-4 scaled recursion after the lean kernel changes
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for h in on off; do
  timeout 300 python bench.py --no-cpu-baseline --l2-hint $h 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('l2-hint=$h', round(d['value']), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms'].items()}, d['clocks'], (d.get('parity_vs_reference') or {}).get('identical'))"
done
done
