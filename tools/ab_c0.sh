cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/c0_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/c0_tests.log
for rec in scaled exact scaled exact; do
  timeout 300 python bench.py --config 0 --recursion $rec --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$rec', round(d['value']), round(d['e2e']['value']), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()}, d['fused_synth'])"
done
