# A/B: programmatic dependent launch of the config-0 latency recursion (default) vs ordinary launch (exp/nopdl.so)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cluster.py -q -m gpu -x > gpurun_out/pdl_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/pdl_tests.log
run() { lib=$1; shift; FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config 0 --steps 300 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('${lib:-pdl}', round(d['value']), round(d['e2e']['value']), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()})"; }
for rep in 1 2 3; do
  run exp/nopdl.so
  run ""
done
