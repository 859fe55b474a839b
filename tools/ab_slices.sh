# A/B: digit planes of the config-4 initial products (FASE_PRODUCT_SLICES)
cd $GRAFT_REPO_ROOT
timeout 600 python tools/probes/product_slices.py > gpurun_out/slices_probe.log 2>&1; echo probe=$?; cat gpurun_out/slices_probe.log | tail -4
for s in 8 7 6 8 7 6; do
  FASE_PRODUCT_SLICES=$s timeout 300 python bench.py --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/ab_s$s.log 2>&1; echo "s=$s rc=$?"
  tail -1 gpurun_out/ab_s$s.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['stage_ms'], d['parity_vs_reference'], d['clocks']['sm_mhz'])"
done
