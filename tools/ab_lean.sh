# A/B: scaled-recursion critical-path trims (FASE_SCALED_LEAN bits; default build = 3)
cd $GRAFT_REPO_ROOT
run() { lib=$1; c=$2; shift 2; FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config $c --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('${lib:-lean3}', 'c$c', '$*', round(d['value']), round(d['ms_per_step'],4), round((d.get('roofline') or {}).get('ms_per_launch',0),4), (d.get('parity_vs_reference') or {}).get('identical'), (d.get('recursion_agreement') or {}).get('blocks_identical_selections'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch_parity.py -q -m gpu -x > gpurun_out/lean_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/lean_tests.log
for rep in 1 2; do
for lib in exp/lean0.so exp/lean1.so exp/lean2.so ""; do
  run "$lib" 4
  run "$lib" 1 --steps 50 --warmup 3
done
done
