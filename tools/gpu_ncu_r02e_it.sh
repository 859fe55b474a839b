# source-level ncu capture of the config-4 integer-key scaled recursion (one launch)
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fase_iterate_kernel" -s 3 -c 1 \
  --metrics lts__t_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_op_read.sum,smsp__inst_executed.sum,l1tex__m_xbar2l1tex_read_bytes.sum \
  -o gpurun_out/prof_r02e_c4it $CMD > gpurun_out/ncu_it.log 2>&1; echo it=$?
