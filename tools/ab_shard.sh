# one rank's shard of the c4 / c1 batch at N = 2 / 4 / 8 on one GPU: products path per size
cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py --no-cpu-baseline "$@" 2>gpurun_out/shard_err.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('$*', round(d['value']), round(d['ms_per_step'],4), d['products'], d['recursion'], {k: round(v,4) for k,v in d['stage_ms'].items()}, pv.get('identical'), pv.get('blocks_checked'), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/shard_err.log; }
for b in 512 1024 2048; do
  for p in auto ozaki gemm; do run --blocks $b --products $p --steps 30 --warmup 3; done
done
for b in 128 256 512; do run --config 1 --blocks $b --steps 50 --warmup 3; done
