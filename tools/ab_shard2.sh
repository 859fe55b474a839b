# after the Ozaki threshold change: GPU suite + c4 shard sizes (N = 16 / 8 / 4 / 2 / 1 per-rank batches)
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/shard2_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/shard2_tests.log
run() { timeout 300 python bench.py --no-cpu-baseline "$@" 2>gpurun_out/shard_err.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('$*', round(d['value']), round(d['ms_per_step'],4), d['products'], d['recursion'], {k: round(v,4) for k,v in d['stage_ms'].items()}, pv.get('identical'), pv.get('blocks_checked'), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/shard_err.log; }
for b in 256 512; do
  for p in auto gemm; do run --blocks $b --products $p --steps 30 --warmup 3; done
done
for b in 1024 2048; do run --blocks $b --steps 30 --warmup 3; done
run --steps 30 --warmup 3
