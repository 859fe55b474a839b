# config 2 (chunked exact): 128 x 36 (4 warps) vs the default 256 x 18; config 3 for reference
cd $GRAFT_REPO_ROOT
run() { env "$@" timeout 300 python bench.py --config 2 --steps 10 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('$*', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), round(d['roofline']['ms_per_launch'],4), pv.get('identical'), (pv.get('all_blocks_selections') or {}).get('identical'))"; }
for rep in 1 2; do
  run X=1
  run FASE_ITERATE_VARIANT=128x36
done
