# A/B: division-free staging loops of the separable products (default) vs the previous build (exp/olddiv.so)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_transform.py tests/test_gpu_conceal.py -q -m gpu -x > gpurun_out/sepdiv_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/sepdiv_tests.log
run() { lib=$1; c=$2; shift 2; FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config $c --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('${lib:-new}', 'c$c', round(d['value']), round(d['e2e']['value']), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()}, (d.get('parity_vs_reference') or {}).get('identical'))"; }
for rep in 1 2; do
for lib in exp/olddiv.so ""; do
  run "$lib" 0 --steps 300 --warmup 5
  run "$lib" 1 --steps 50 --warmup 3
done
done
