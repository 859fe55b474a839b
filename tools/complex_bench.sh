# complex-dictionary benches on config-1 geometry (+ variant override sweep)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_complex.py -x -q -m gpu > gpurun_out/gpu_complex.log 2>&1; echo tests=$?; tail -1 gpurun_out/gpu_complex.log
for spec in dft union:dft+bdft; do
  for v in "" 256x9x3; do
    FASE_ITERATE_COMPLEX_VARIANT=$v python bench.py --config 1 --dict $spec --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cx.log 2>&1; echo "$spec variant=$v rc=$?"
    tail -1 gpurun_out/bench_cx.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['stage_ms'], 'frac', round(d['roofline']['frac'],3), 'gram_ms', round(d['gram_ms'],2), 'e2e', round(d['e2e']['value']))"
  done
done
