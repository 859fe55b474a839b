cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_all.log 2>&1; echo tests=$?; tail -15 gpurun_out/gpu_all.log
for c in 3 2; do
timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/b$c.log 2>&1; echo "c$c rc=$?"; tail -1 gpurun_out/b$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], round(d['e2e']['value']), d['parity_vs_reference'])"
done
