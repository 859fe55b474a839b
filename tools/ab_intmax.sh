# A/B: integer high-word running max in the scaled recursion (FASE_SCALED_LEAN bit 32, exp/intmax.so) vs default
cd $GRAFT_REPO_ROOT
run() { lib=$1; c=$2; shift 2; FASE_B200_LIB=${lib:-paper_2204_14194_b200/libfase_b200.so} timeout 300 python bench.py --config $c --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pv=d.get('parity_vs_reference') or {}
print('${lib:-default}', 'c$c', '$*', round(d['value']), round(d['ms_per_step'],4), round((d.get('roofline') or {}).get('ms_per_launch',0),4), pv.get('identical'), (pv.get('all_blocks_selections') or {}).get('identical'), (d.get('recursion_agreement') or {}).get('blocks_identical_selections'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
FASE_B200_LIB=exp/intmax.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch_parity.py tests/test_gpu_complex.py tests/test_gpu_cluster.py -q -m gpu -x > gpurun_out/intmax_tests.log 2>&1; echo tests_intmax=$?; tail -3 gpurun_out/intmax_tests.log
for rep in 1 2; do
for lib in exp/intmax.so ""; do
  run "$lib" 4
  run "$lib" 1 --steps 50 --warmup 3
done
done
run exp/intmax.so 0 --steps 200 --warmup 5
run "" 0 --steps 200 --warmup 5
