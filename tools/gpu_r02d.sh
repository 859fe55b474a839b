# re-entry check (round 2, third session): full GPU suite, smoke, default bench
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_all.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_default.log | cut -c1-600
