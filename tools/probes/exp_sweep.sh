# recursion-kernel ablations: 0 = library, 1 = no D loads, 2 = no row staging, 3 = no tie pass
for e in 0 1 2 3; do
  if [ $e = 0 ]; then unset FASE_B200_LIB; else export FASE_B200_LIB=$PWD/tools/probes/libexp$e.so; fi
  python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('exp$e', d['stage_ms']['iterate'])"
done
