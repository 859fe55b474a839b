cd $GRAFT_REPO_ROOT
for g in 8 2 4 16 32 64 8; do
  FASE_OZAKI_GROUP_M=$g timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('group_m=$g', round(d['value']), {k: round(v,4) for k,v in d['stage_ms'].items()}, d['clocks']['sm_mhz'])"
done
