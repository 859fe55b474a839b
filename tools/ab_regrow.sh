cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cluster.py tests/test_gpu_complex.py -q -m gpu -x > gpurun_out/regrow_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/regrow_tests.log
for lib in exp/tma0.so "" exp/tma0.so ""; do
  for rec in scaled exact; do
  FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config 0 --recursion $rec --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('${lib:-default(regrow)}', '$rec', round(d['value']), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()})"
  done
done
for lib in exp/tma0.so ""; do FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} FASE_CLUSTER=0 python tools/probes/cluster_probe.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('${lib:-regrow}', d['config'], d['blocks'], d['recursion'], round(d['us_per_iter']['single'],3))"; done
