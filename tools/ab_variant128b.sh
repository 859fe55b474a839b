# after making 128 x 64 the capacity-8192 default: GPU suite + config 4 default vs the old 256 x 32
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/v128_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/v128_tests.log
run() { env "$@" timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('$*', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), {k: round(v,4) for k,v in d['stage_ms'].items()}, pv.get('identical'), (pv.get('all_blocks_selections') or {}).get('identical'), d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
  run X=1
  run FASE_SCALED_VARIANT=256x32x2
done
