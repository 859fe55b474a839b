# A/B: fused update in the scaled recursion (FASE_SCALED_LEAN=5 build) vs default (1)
cd $GRAFT_REPO_ROOT
run() { lib=$1; c=$2; shift 2; FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config $c --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('${lib:-lean1}', 'c$c', '$*', round(d['value']), round(d['ms_per_step'],4), round((d.get('roofline') or {}).get('ms_per_launch',0),4), pv.get('identical'), pv.get('near_tie'), pv.get('max_coef_rel_dev'), (pv.get('all_blocks_selections') or {}).get('identical'), (d.get('recursion_agreement') or {}).get('blocks_identical_selections'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do
for lib in exp/lean5.so exp/lean1.so ""; do
  run "$lib" 4
  run "$lib" 1 --steps 50 --warmup 3
done
done
