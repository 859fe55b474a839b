cd $GRAFT_REPO_ROOT
timeout 300 python tools/probes/split_timing.py 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ozaki_split_sparse" -s 3 -c 1 \
  -o gpurun_out/prof_split_sparse python tools/probes/split_timing.py > gpurun_out/ncu_split.log 2>&1; echo ncu=$?
