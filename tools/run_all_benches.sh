# round-end evidence: every config's bench line (CPU baseline included), the
# complex default dictionary on config-1 geometry, then ncu (launch list of
# config 1, full captures of the config-1 kernels, the config-4 tcgen05 Ozaki
# products and the complex recursion)
mkdir -p gpurun_out/benches
python bench.py > gpurun_out/benches/c1.json 2> gpurun_out/benches/c1.err; echo c1=$?
python bench.py --config 0 --steps 50 --warmup 5 --cpu-seconds 8 > gpurun_out/benches/c0.json 2> gpurun_out/benches/c0.err; echo c0=$?
for c in 4 3 2; do
  python bench.py --config $c --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/benches/c$c.json 2> gpurun_out/benches/c$c.err; echo c$c=$?
done
python bench.py --config 1 --dict dft --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/benches/c1_dft.json 2> gpurun_out/benches/c1_dft.err; echo c1dft=$?
python bench.py --config 1 --dict union:dft+bdft --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/benches/c1_dftbdft.json 2> gpurun_out/benches/c1_dftbdft.err; echo c1dftbdft=$?
python bench.py --config 1 --recursion exact --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/benches/c1_exact.json 2> gpurun_out/benches/c1_exact.err; echo c1exact=$?
python bench.py --config 4 --recursion exact --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/benches/c4_exact.json 2> gpurun_out/benches/c4_exact.err; echo c4exact=$?
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/benches/c1_reference.json 2> gpurun_out/benches/c1_reference.err; echo ref=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01g.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:"fase_iterate|sep_products|weigh|synth_paste" -s 5 -c 5 -o gpurun_out/prof_r01_c1g python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ozaki_gemm" -s 2 -c 1 -o gpurun_out/prof_r01_c4g_products python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu4.log 2>&1; echo ncu4=$?
ncu --set full --clock-control none --import-source on -k regex:"fase_iterate" -c 1 -o gpurun_out/prof_r01_c4g_iterate python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu4b.log 2>&1; echo ncu4b=$?
python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fase_iterate" -c 1 -o gpurun_out/prof_r01_c2g python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2b.log 2>&1; echo ncu2b=$?
ncu --set full --clock-control none --import-source on -k regex:"iterate_complex|sep_products_complex" -s 2 -c 2 -o gpurun_out/prof_r01_dftg python bench.py --config 1 --dict dft --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu5.log 2>&1; echo ncu5=$?
python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fase_iterate" -c 1 -o gpurun_out/prof_r01_c3g python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3b.log 2>&1; echo ncu3b=$?
# gpurun brings back at most 64 MiB: export the raw pages, drop the reports
for r in gpurun_out/prof_r01_*g*.ncu-rep; do ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" && rm -f "$r"; done
