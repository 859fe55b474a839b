# source-level ncu capture of the config-4 scaled recursion (one launch)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fase_iterate_kernel" -s 3 -c 1 \
  --metrics lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum,smsp__inst_executed.sum \
  -o gpurun_out/prof_r02_c4src $CMD > gpurun_out/ncu_c4src.log 2>&1; echo c4=$?
