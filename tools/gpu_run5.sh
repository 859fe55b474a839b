cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/sanitize_cases.py > gpurun_out/checked_default.log 2>&1; echo default=$?; cat gpurun_out/checked_default.log | tail -14
FASE_B200_LIB=exp/bounds.so timeout 900 python tools/sanitize_cases.py > gpurun_out/checked_bounds.log 2>&1; echo bounds=$?; tail -14 gpurun_out/checked_bounds.log
FASE_B200_LIB=exp/bounds.so timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/checked_pytest.log 2>&1; echo pytest_bounds=$?; tail -3 gpurun_out/checked_pytest.log
