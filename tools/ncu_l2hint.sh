cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
M=gpu__time_duration.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum
$CMD > gpurun_out/plain_h.log 2>&1 && \
FASE_L2_HINT=1 ncu --clock-control none --metrics $M -k regex:fase_iterate_kernel -s 3 -c 1 --csv --log-file gpurun_out/r02_l2hint_on.csv $CMD > gpurun_out/ncu_h1.log 2>&1; echo on=$?
FASE_L2_HINT=0 ncu --clock-control none --metrics $M -k regex:fase_iterate_kernel -s 3 -c 1 --csv --log-file gpurun_out/r02_l2hint_off.csv $CMD > gpurun_out/ncu_h0.log 2>&1; echo off=$?
for f in on off; do grep -v "^==" gpurun_out/r02_l2hint_$f.csv | python -c "
import csv,sys
for r in csv.DictReader(sys.stdin): print('$f', r['Metric Name'], r['Metric Value'], r['Metric Unit'])"; done
