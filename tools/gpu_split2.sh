cd $GRAFT_REPO_ROOT
timeout 300 python tools/probes/split_timing.py 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_transform.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
for i in 1 2; do
timeout 300 python bench.py --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/b_split.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/b_split.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['parity_vs_reference']; print(round(d['value']), round(d['e2e']['value']), d['stage_ms'], d['clocks']['sm_mhz'], {k:p[k] for k in ('identical','near_tie','failure','max_coef_rel_dev','max_lost_rel_dev')}, p['all_blocks_selections'])"
done
