# A/B: costliest-first dispatch of the frame recursion (FASE_BLOCK_ORDER) + the GPU suite
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/order_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/order_tests.log
run() { o=$1; c=$2; shift 2; FASE_BLOCK_ORDER=$o timeout 300 python bench.py --config $c --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('order=$o', 'c$c', '$*', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), round((d.get('roofline') or {}).get('ms_per_launch',0),4), pv.get('identical'), (pv.get('all_blocks_selections') or {}).get('identical'), d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
for o in 0 1; do
  run $o 2 --steps 10 --warmup 2
  run $o 3 --steps 5 --warmup 2
  run $o 2 --dict dft --steps 10 --warmup 2
done
done
