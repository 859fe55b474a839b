cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_complex.py -x -q 2>&1 | tail -3
for spec in union:dft+bdft union:dct+dft; do
for P in 0 1; do
  FASE_ITERATE_PAIR=$P python bench.py --config 1 --dict $spec --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cpair_$P.log 2>&1; echo "$spec pair=$P rc=$?"
  tail -1 gpurun_out/cpair_$P.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['stage_ms'], 'e2e', round(d['e2e']['value']))"
done; done
