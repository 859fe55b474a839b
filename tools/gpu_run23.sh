cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_transform.py -q -m gpu -x > gpurun_out/sep_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/sep_tests.log
for c in 0 1; do
timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('c$c', round(d['value']), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stage_ms'].items()})"
done
