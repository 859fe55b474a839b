# full check: GPU suite, smoke(), default bench (driver's command), reference arm
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/r02b
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02b/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02b/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02b/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/r02b/smoke.log
python bench.py > gpurun_out/r02b/c4.json 2> gpurun_out/r02b/c4.err; echo c4=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02b/c4_reference.json 2> gpurun_out/r02b/c4_reference.err; echo ref=$?
for f in gpurun_out/r02b/*.json; do echo "$f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d.get('e2e',{}).get('value',0)), d.get('clocks',{}).get('sm_mhz'), (d.get('parity_vs_reference') or {}).get('identical'))" 2>/dev/null)"; done
