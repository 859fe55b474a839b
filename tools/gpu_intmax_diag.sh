# diagnosis of the integer-max scaled recursion: source-level ncu captures of both builds
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
for lib in exp/intmax.so paper_2204_14194_b200/libfase_b200.so; do
  tag=$(basename $lib .so)
  FASE_B200_LIB=$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fase_iterate_kernel" -s 3 -c 1 \
    -o gpurun_out/prof_src_$tag $CMD > gpurun_out/ncu_$tag.log 2>&1; echo ncu_$tag=$?
done
