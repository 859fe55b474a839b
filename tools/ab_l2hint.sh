cd $GRAFT_REPO_ROOT
for c in 4 1; do
  for h in 1 0; do
    FASE_L2_HINT=$h timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline 2>gpurun_out/ab_err.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('c$c hint=$h', round(d['value']), {k: round(v,4) for k,v in d['stage_ms'].items()}, d['clocks']['sm_mhz'], d['clocks']['reasons'], (d.get('l2_hint') or {}).get('hot_rows'), round((d.get('l2_hint') or {}).get('hot_share_of_tuning_selections',0),3), d['parity_vs_reference']['identical'])"
  done
done
tail -3 gpurun_out/ab_err.log
