cd $GRAFT_REPO_ROOT
for i in 1 2; do
  for rec in scaled exact; do
  timeout 300 python bench.py --config 0 --recursion $rec --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$rec', round(d['value']), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()}, d['fused_synth'])"
  done
done
FASE_CLUSTER=0 python tools/probes/cluster_probe.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['blocks'], d['recursion'], round(d['us_per_iter']['single'],3))"
