cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1; echo plain=$?; tail -15 gpurun_out/sanitize_plain.log
SAN_TIMEOUT=1200 bash tools/sanitize.sh
