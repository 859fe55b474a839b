cd $GRAFT_REPO_ROOT
run() { label=$1; shift; env "$@" timeout 300 python bench.py --config 1 --dict dft --steps 20 --warmup 3 --no-cpu-baseline --recursion $REC 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$label', round(d['value']), round(d['ms_per_step'],3), {k: round(v,4) for k,v in d['stage_ms'].items()}, (d.get('parity_vs_reference') or {}).get('identical'))"; }
for rep in 1 2; do
REC=exact run exact-default X=1
REC=exact run exact-256x9x4 FASE_ITERATE_COMPLEX_VARIANT=256x9x4
REC=scaled run scaled-default X=1
REC=scaled run scaled-256x9x4 FASE_COMPLEX_SCALED_VARIANT=256x9x4
done
