cd $GRAFT_REPO_ROOT
for lib in exp/ef2.so "" exp/ef2.so ""; do
  for c in 2 3; do
    FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config $c --steps 10 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('${lib:-default(evict_first)}', 'c$c', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['ms_per_launch'],3), d['parity_vs_reference']['identical'], d['clocks']['sm_mhz'])"
  done
done
