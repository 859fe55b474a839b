# A/B the scaled recursion builds (exp/*.so) on configs 4 and 1: stage split
cd $GRAFT_REPO_ROOT
for lib in "" ${LIBS:-exp/seg4.so exp/seg8.so exp/ch2.so exp/ch2seg4.so}; do
  for c in ${CONFIGS:-4 1}; do
    FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('${lib:-default}', 'c$c', round(d['value']), {k: round(v,4) for k,v in d['stage_ms'].items()}, d['parity_vs_reference']['identical'] if d.get('parity_vs_reference') else None)"
  done
done
