# A/B: integer keys on the 18-element shape with re-derived output rows (exp/intmax18.so), output rows alone on config 4 (exp/outrow.so), default
cd $GRAFT_REPO_ROOT
run() { lib=$1; c=$2; shift 2; FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config $c --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('${lib:-default}', 'c$c', '$*', round(d['value']), round(d['ms_per_step'],4), round((d.get('roofline') or {}).get('ms_per_launch',0),4), pv.get('identical'), (pv.get('all_blocks_selections') or {}).get('identical'), (d.get('recursion_agreement') or {}).get('blocks_identical_selections'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
FASE_B200_LIB=exp/intmax18.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch_parity.py -q -m gpu -x > gpurun_out/intmax18_tests.log 2>&1; echo tests_intmax18=$?; tail -2 gpurun_out/intmax18_tests.log
for rep in 1 2; do
  run exp/intmax18.so 1 --steps 50 --warmup 3
  run "" 1 --steps 50 --warmup 3
  run exp/outrow.so 4
  run "" 4
done
