# complex recursion residency on the dft config-1 geometry: default vs four CTAs/SM
for v in "" 256x9x4 128x18x4; do
  FASE_ITERATE_COMPLEX_VARIANT=$v python bench.py --config 1 --dict dft --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cm_$v.json 2> gpurun_out/cm_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/cm_$v.json').read().strip().splitlines()[-1]); print('variant=$v', round(d['value']), round(d['stage_ms']['iterate'],4))"
done
