# config 1: scaled recursion 128 x 36 (4 warps) vs the default 256 x 18, four CTAs per SM
cd $GRAFT_REPO_ROOT
run() { env "$@" timeout 300 python bench.py --config 1 --steps 50 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('$*', round(d['value']), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms'].items()}, pv.get('identical'), d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
  run X=1
  run FASE_SCALED_VARIANT=128x36x4
  run FASE_SCALED_VARIANT=256x18x3
done
