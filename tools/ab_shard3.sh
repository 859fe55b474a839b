# third session: one rank's shard of config 4 on the final kernels (N = 8 / 4 / 2 / 1 per-rank batches)
cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py --no-cpu-baseline "$@" 2>gpurun_out/shard_err.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('$*', round(d['value']), round(d['ms_per_step'],4), d['products'], d['recursion'], {k: round(v,4) for k,v in d['stage_ms'].items()}, pv.get('identical'), pv.get('blocks_checked'), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/shard_err.log; }
for b in 512 1024 2048; do run --blocks $b --steps 30 --warmup 3; done
run --steps 30 --warmup 3
