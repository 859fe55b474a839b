# complex-dictionary benches on config-1 geometry
cd $GRAFT_REPO_ROOT
for spec in dft union:dft+bdft union:dct+dft; do
  python bench.py --config 1 --dict $spec --steps 10 --warmup 3 ${CPU_ARGS:---no-cpu-baseline} > gpurun_out/bench_cx_$(echo $spec|tr ':+' '__').log 2>&1; echo "$spec rc=$?"
  tail -1 gpurun_out/bench_cx_$(echo $spec|tr ':+' '__').log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['products'], d['stage_ms'], 'frac', round(d['roofline']['frac'],3), 'gram_ms', round(d['gram_ms'],2), 'fft_gram_ms', d['fft_gram_ms'], 'e2e', round(d['e2e']['value']), 'cpu', (d['cpu_baseline'] or {}).get('value'))"
done
