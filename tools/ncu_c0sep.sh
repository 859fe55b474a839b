# source-level ncu capture of the config-0 separable products kernel (one block)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config 0 --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_c0.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sep_products" -s 5 -c 1 \
  -o gpurun_out/prof_r02b_c0sep $CMD > gpurun_out/ncu_c0sep.log 2>&1; echo c0sep=$?
