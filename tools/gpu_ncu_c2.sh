cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config 2 --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fase_iterate_kernel" -s 2 -c 1 \
  --metrics lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum,smsp__inst_executed.sum \
  -o gpurun_out/prof_r02_c2 $CMD > gpurun_out/ncu_c2.log 2>&1; echo c2=$?
CMD3="python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline"
$CMD3 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fase_iterate_kernel" -s 2 -c 1 \
  --metrics lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum,smsp__inst_executed.sum \
  -o gpurun_out/prof_r02_c3 $CMD3 > gpurun_out/ncu_c3.log 2>&1; echo c3=$?
