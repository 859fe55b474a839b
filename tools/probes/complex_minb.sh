# complex recursion at 3 CTAs/SM: timing with a build whose exact |z| is replaced
# by a call-free stand-in (upper bound of what call-free exact arithmetic buys)
cd $GRAFT_REPO_ROOT
for lib in "" tools/probes/exp_lib/libfase_b200_fakeabs.so; do
  for v in "" 256x9x3; do
    FASE_B200_LIB=$lib FASE_ITERATE_COMPLEX_VARIANT=$v python bench.py --config 1 --dict dft --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cm.log 2>&1
    echo "lib=${lib:-default} variant=${v:-default}: $(tail -1 gpurun_out/cm.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['stage_ms']['iterate'])")"
  done
done
