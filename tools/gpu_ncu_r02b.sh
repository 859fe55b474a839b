# round-2 (second session) ncu captures after the lean scaled recursion: c4 launch list, --set full of the recursion / products / synthesis, L2 probe counters
# the recursion / products / synthesis kernels, and the L2 probe's counters
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/l2_probe tools/probes/l2_probe.cu
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fase_iterate_kernel|ozaki_gemm|synth_paste" -s 6 -c 3 \
  --metrics lts__t_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_op_read.sum,smsp__inst_executed.sum \
  -o gpurun_out/prof_r02b_c4 $CMD > gpurun_out/ncu_full.log 2>&1; echo full=$?
gpurun_out/l2_probe > gpurun_out/l2_plain.json 2>&1 && \
ncu --clock-control none --metrics gpu__time_duration.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum --csv --log-file gpurun_out/r02b_l2probe_ncu.csv gpurun_out/l2_probe > gpurun_out/ncu_l2.log 2>&1; echo l2=$?
ls -la gpurun_out/*.ncu-rep
