# all GPU tests + quick benches of the given configs
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_all.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_all.log
for c in ${CONFIGS:-1}; do
  python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline > gpurun_out/b$c.log 2>&1; echo "c$c rc=$?"
  tail -1 gpurun_out/b$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d.get('products'), d.get('stage_ms'), (d.get('roofline_init') or {}).get('frac'))"
done
