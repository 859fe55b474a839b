cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_complex.py tests/test_gpu_batch_parity.py tests/test_gpu_conceal.py -q -m gpu -x > gpurun_out/cplx_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/cplx_tests.log
for spec in dft union:dft+bdft union:dct+dft; do
timeout 300 python bench.py --config 1 --dict $spec --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$spec', d['recursion'], round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],3), {k: round(v,4) for k,v in d['stage_ms'].items()}, (d.get('parity_vs_reference') or {}).get('identical'))"
done
