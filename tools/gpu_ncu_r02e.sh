# round-2 (third session) ncu captures after the integer-key scaled recursion: c4 launch list, --set full of the recursion / products / synthesis kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fase_iterate_kernel|ozaki_gemm|ozaki_split" -s 6 -c 4 \
  --metrics lts__t_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_op_read.sum,smsp__inst_executed.sum,l1tex__m_xbar2l1tex_read_bytes.sum \
  -o gpurun_out/prof_r02e_c4 $CMD > gpurun_out/ncu_full.log 2>&1; echo full=$?
ls -la gpurun_out/*.ncu-rep
