cd $GRAFT_REPO_ROOT
for g in 1 4 8 16 32; do echo "group_m=$g"; FASE_OZAKI_GROUP_M=$g timeout 120 python tools/probes/ozaki_slices.py 2>&1 | grep "s=8"; done
