# Ozaki synthesis: new GPU tests, Ozaki-path tests, then config-4 A/B (paste vs ozaki synthesis)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_transform.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/t_synth.log 2>&1; echo tests=$?; tail -3 gpurun_out/t_synth.log
for m in paste auto paste auto; do
  FASE_SYNTH=$m timeout 300 python bench.py --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/ab_synth_$m.log 2>&1; echo "synth=$m rc=$?"
  tail -1 gpurun_out/ab_synth_$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['parity_vs_reference']; print(round(d['value']), round(d['e2e']['value']), d['synthesis'], d['stage_ms'], d['clocks']['sm_mhz'], {k:p[k] for k in ('identical','near_tie','failure','max_coef_rel_dev','max_lost_rel_dev')}, p['all_blocks_selections'])"
done
