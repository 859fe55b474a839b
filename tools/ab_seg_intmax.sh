# A/B on the integer-key config-4 recursion: staged-row segments 2 / 3 (default) / 4, L2 residency hint
cd $GRAFT_REPO_ROOT
run() { lib=$1; c=$2; shift 2; FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config $c --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('${lib:-default}', 'c$c', '$*', round(d['value']), round(d['ms_per_step'],4), round((d.get('roofline') or {}).get('ms_per_launch',0),4), pv.get('identical'), (pv.get('all_blocks_selections') or {}).get('identical'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do
  run exp/seg2.so 4
  run exp/seg4.so 4
  run "" 4
  run "" 4 --l2-hint on
done
