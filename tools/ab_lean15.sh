# A/B: D prefetch after the block max (bit 2) on top of the default scaled-recursion trims (13)
cd $GRAFT_REPO_ROOT
run() { lib=$1; c=$2; shift 2; FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config $c --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('${lib:-lean13}', 'c$c', '$*', round(d['value']), round(d['ms_per_step'],4), round((d.get('roofline') or {}).get('ms_per_launch',0),4), pv.get('identical'), d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
for lib in exp/lean15.so ""; do
  run "$lib" 1 --steps 50 --warmup 3
  run "$lib" 4
  run "$lib" 1 --dict dft --steps 20 --warmup 3
done
done
