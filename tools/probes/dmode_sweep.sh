# recursion variants for config 1: default vs D through L1 (3 or 4 CTAs/SM)
cd $GRAFT_REPO_ROOT
for v in "" 256x18x3x2 256x18x4x2; do
  FASE_ITERATE_VARIANT=$v python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_v.log 2>&1; echo "variant=$v rc=$?"
  tail -1 gpurun_out/bench_v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['stage_ms'])"
done
