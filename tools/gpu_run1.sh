cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch_parity.py -q -s -m gpu > gpurun_out/batch_parity.log 2>&1; echo tests=$?; grep "batch parity" gpurun_out/batch_parity.log; tail -3 gpurun_out/batch_parity.log
timeout 300 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/b4.log | cut -c1-1500
