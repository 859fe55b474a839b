# every config's bench line (CPU baseline included), then ncu of config 1
mkdir -p gpurun_out/benches
python bench.py > gpurun_out/benches/c1.json 2> gpurun_out/benches/c1.err; echo c1=$?
for c in 0 4 3 2; do
  python bench.py --config $c --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/benches/c$c.json 2> gpurun_out/benches/c$c.err; echo c$c=$?
done
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:"fase_iterate|sep_products|weigh|synth_paste" -s 5 -c 5 -o gpurun_out/prof_r01_c1b python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
