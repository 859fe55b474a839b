# after the tie-quantum gate fix: the integer-key test, the parity suites, smoke, the default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02g
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02g/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02g/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02g/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/r02g/c4.json 2> gpurun_out/r02g/c4.err; echo c4=$?
tail -1 gpurun_out/r02g/c4.json | cut -c1-400
