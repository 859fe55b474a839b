# small-batch separable products with staged factor tables: tests + config 0 / 1 bench
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_transform.py -q -m gpu -x > gpurun_out/sep_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/sep_tests.log
for rep in 1 2; do
  timeout 300 python bench.py --config 0 --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('c0', round(d['value']), round(d['e2e']['value']), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()})"
  timeout 300 python bench.py --config 1 --steps 50 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('c1', round(d['value']), round(d['e2e']['value']), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()})"
done
