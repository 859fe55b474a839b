# A/B: the simplified tie-quantum / threshold arithmetic (default build) vs the previous commit (exp/headq.so)
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/q_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/q_tests.log
run() { lib=$1; c=$2; shift 2; FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config $c --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('${lib:-new}', 'c$c', '$*', round(d['value']), round(d['ms_per_step'],4), round((d.get('roofline') or {}).get('ms_per_launch',0),4), pv.get('identical'), (pv.get('all_blocks_selections') or {}).get('identical'), d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
for lib in exp/headq.so ""; do
  run "$lib" 4
  run "$lib" 1 --steps 50 --warmup 3
  run "$lib" 3 --steps 5 --warmup 2
  run "$lib" 0 --steps 200 --warmup 5
done
done
