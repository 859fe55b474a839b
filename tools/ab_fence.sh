# A/B: the proxy fence before each TMA row refill (FASE_ISSUE_FENCE=0 build in exp/nofence.so)
cd $GRAFT_REPO_ROOT
run() { lib=$1; c=$2; shift 2; FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config $c --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
st=d.get('stage_ms') or {}
print('${lib:-default}', 'c$c', '$*', round(d['value']), round(d['ms_per_step'],4), round((d.get('roofline') or {}).get('ms_per_launch',0),4), (d.get('parity_vs_reference') or {}).get('identical'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do
for lib in exp/nofence.so ""; do
  run "$lib" 0 --steps 200 --warmup 5
  run "$lib" 1 --steps 30 --warmup 3
  run "$lib" 2 --steps 10 --warmup 2
  run "$lib" 3 --steps 5 --warmup 2
  run "$lib" 4 --steps 10 --warmup 3
  run "$lib" 1 --dict dft --steps 20 --warmup 3
done
done
