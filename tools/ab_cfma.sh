# A/B: fused update in the complex scaled recursion (default) vs numpy-order (exp/cfma0.so)
cd $GRAFT_REPO_ROOT
run() { lib=$1; c=$2; shift 2; FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config $c --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('${lib:-default}', 'c$c', '$*', round(d['value']), round(d['ms_per_step'],4), round((d.get('roofline') or {}).get('ms_per_launch',0),4), pv.get('identical'), pv.get('near_tie'), pv.get('max_coef_rel_dev'), (d.get('recursion_agreement') or {}).get('blocks_identical_selections'), d['clocks']['sm_mhz'])"; }
timeout 900 python -m pytest tests/test_gpu_complex.py tests/test_gpu_batch_parity.py -q -m gpu -x > gpurun_out/cfma_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/cfma_tests.log
for rep in 1 2; do
for lib in exp/cfma0.so ""; do
  run "$lib" 1 --dict dft --steps 20 --warmup 3
  run "$lib" 1 --dict union:dft+bdft --steps 10 --warmup 3
done
done
