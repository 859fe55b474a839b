# quick regression check of every BASELINE config (device value and stage split)
cd ${GRAFT_REPO_ROOT:-.}
for c in ${CONFIGS:-1 4 2 3 0}; do
  python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/reg_c$c.log 2>&1
  tail -1 gpurun_out/reg_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c$c', round(d['value']), 'iter_ms', round(d.get('stage_ms', {}).get('iterate') or r.get('ms_per_launch'), 3), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])"
done
