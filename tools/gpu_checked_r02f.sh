# end of round 2, third session (integer-key recursion): the checked build (FASE_BOUNDS) and determinism / operand-integrity cases
# over every kernel family incl. the second session's (streaming recursions, row-panel Gram,
# block order in the frame case), then the GPU suite on the checked build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02f_checked
timeout 900 python tools/sanitize_cases.py > gpurun_out/r02f_checked/checked_default.log 2>&1; echo default=$?; tail -20 gpurun_out/r02f_checked/checked_default.log
FASE_B200_LIB=exp/bounds.so timeout 1200 python tools/sanitize_cases.py > gpurun_out/r02f_checked/checked_bounds.log 2>&1; echo bounds=$?; tail -20 gpurun_out/r02f_checked/checked_bounds.log
FASE_B200_LIB=exp/bounds.so timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02f_checked/checked_pytest.log 2>&1; echo pytest_bounds=$?; tail -3 gpurun_out/r02f_checked/checked_pytest.log
