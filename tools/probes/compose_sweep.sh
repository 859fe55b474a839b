# frame configs with and without precomposed base tables
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -x -q -k "frame_engine" 2>&1 | tail -2
for c in 2 3; do for m in none singles pairs; do
  python bench.py --config $c --compose $m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cmp_${c}_$m.log 2>&1; echo "c$c $m rc=$?"
  tail -1 gpurun_out/cmp_${c}_$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']), round(d['ms_per_step'],3), 'iter_ms', round(r['ms_per_launch'],3), 'rows', round(d['config']['mean_rows_per_iteration'],2), 'e2e', round(d['e2e']['value']), 'build_s', round(d['table_build_s'],2))"
done; done
