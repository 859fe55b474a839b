# config 0 (one block): scaled vs exact recursion after the lean scaled kernel
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for rec in exact scaled; do
  timeout 300 python bench.py --config 0 --recursion $rec --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$rec', round(d['value']), round(d['e2e']['value']), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()}, d['fused_synth'])"
done
done
