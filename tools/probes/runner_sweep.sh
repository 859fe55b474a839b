# chunked recursion: runner-up L2 prefetch on / off (configs 2 and 3)
for c in 2 3; do
  for rp in 1 0; do
    FASE_RUNNER_PREFETCH=$rp python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rp_c${c}_$rp.json 2> gpurun_out/rp_c${c}_$rp.err
    python -c "import json; d=json.loads(open('gpurun_out/rp_c${c}_$rp.json').read().strip().splitlines()[-1]); print('c$c runner=$rp', round(d['value']), round(d['roofline']['ms_per_launch'],3))"
  done
done
