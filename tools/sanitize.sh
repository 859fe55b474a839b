# compute-sanitizer (memcheck, racecheck, synccheck) over every kernel family
# (tools/sanitize_cases.py); logs under gpurun_out/sanitize_<tool>.log
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout ${SAN_TIMEOUT:-1500} $CS --tool $tool $extra --print-limit 50 --target-processes all \
    python tools/sanitize_cases.py ${CASE:+--case $CASE} > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|^case " gpurun_out/sanitize_$tool.log | tail -20
done
