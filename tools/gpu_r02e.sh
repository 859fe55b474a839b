# integer-max default build: new test first, then the full GPU suite and the config-4 / config-1 lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02e
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "integer_max or scaled" > gpurun_out/r02e/intmax_test.log 2>&1; echo intmax_tests=$?; tail -5 gpurun_out/r02e/intmax_test.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02e/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02e/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02e/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/r02e/c4.json 2> gpurun_out/r02e/c4.err; echo c4=$?
python bench.py --config 1 --cpu-seconds 8 > gpurun_out/r02e/c1.json 2> gpurun_out/r02e/c1.err; echo c1=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02e/c4_reference.json 2> gpurun_out/r02e/c4_reference.err; echo ref=$?
for f in gpurun_out/r02e/*.json; do echo "$f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d.get('e2e',{}).get('value',0)), d.get('stage_ms'), d.get('clocks',{}).get('sm_mhz'), (d.get('parity_vs_reference') or {}))" 2>/dev/null)"; done
