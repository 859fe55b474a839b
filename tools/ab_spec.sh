cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cluster.py -q -m gpu -x > gpurun_out/spec_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/spec_tests.log
for lib in exp/spec0.so "" exp/spec0.so ""; do
  for rec in scaled exact; do
    FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config 0 --recursion $rec --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('${lib:-default(spec3)}', '$rec', round(d['value']), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()}, d['clocks']['sm_mhz'])"
  done
done
FASE_CLUSTER=0 python tools/probes/cluster_probe.py 2>&1 | head -8
