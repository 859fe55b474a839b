cd $GRAFT_REPO_ROOT
timeout 300 python tools/probes/split_timing.py 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_transform.py -x -q -m gpu -k "ozaki or synth" 2>&1 | tail -3
