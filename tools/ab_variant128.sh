# A/B: config-4 scaled recursion shape 128 x 64 (4 warps, 255 registers, 2 CTAs/SM) vs the default 256 x 32
cd $GRAFT_REPO_ROOT
run() { env "$@" timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('$*', round(d['value']), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms'].items()}, pv.get('identical'), (pv.get('all_blocks_selections') or {}).get('identical'), d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
  run X=1
  run FASE_SCALED_VARIANT=128x64x2
  run FASE_SCALED_VARIANT=128x64x3
done
