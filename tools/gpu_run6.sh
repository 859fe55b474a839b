cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_parity.py tests/test_gpu_conceal.py -x -q -m gpu > gpurun_out/cluster_tests.log 2>&1; echo tests=$?; tail -5 gpurun_out/cluster_tests.log
for cl in 4 0; do
  FASE_CLUSTER=$cl timeout 300 python bench.py --config 0 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/b0_cl$cl.log 2>&1; echo "c0 cluster=$cl rc=$?"
  tail -1 gpurun_out/b0_cl$cl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['stage_ms'], d['fused_synth'], d['e2e']['value'])"
  FASE_CLUSTER=$cl timeout 300 python bench.py --config 0 --recursion exact --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/b0x_cl$cl.log 2>&1; echo "c0 exact cluster=$cl rc=$?"
  tail -1 gpurun_out/b0x_cl$cl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['stage_ms'], d['fused_synth'])"
done
