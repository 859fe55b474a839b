cd $GRAFT_REPO_ROOT
rm -f gpurun_out/batch_parity.json
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_all.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b4_r19.log 2>&1; echo bench=$?
tail -1 gpurun_out/b4_r19.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['parity_vs_reference'], d['e2e_dropin'])"
