# time the recursion variants: default vs alternatives (config 1 and 3)
for v in default 128x36; do
  if [ "$v" = default ]; then unset FASE_ITERATE_VARIANT; else export FASE_ITERATE_VARIANT=$v; fi
  python bench.py --config 1 --steps 10 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', '$v', d['stage_ms'])"
done
for v in default 256x8; do
  if [ "$v" = default ]; then unset FASE_ITERATE_VARIANT; else export FASE_ITERATE_VARIANT=$v; fi
  python bench.py --config 3 --steps 3 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', '$v', d['ms_per_step'], d['roofline']['ms_per_launch'])"
done
