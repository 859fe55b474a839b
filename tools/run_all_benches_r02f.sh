# round-2 (third session, final) evidence: GPU tests, every config's bench line
# (CPU baseline included), complex dictionaries, exact recursions, reference arm
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/benches_r02f
rm -f gpurun_out/batch_parity.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/benches_r02f/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/benches_r02f/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/benches_r02f/pytest_gpu.log
python bench.py > gpurun_out/benches_r02f/c4.json 2> gpurun_out/benches_r02f/c4.err; echo c4=$?
python bench.py --config 0 --steps 200 --warmup 5 --cpu-seconds 8 > gpurun_out/benches_r02f/c0.json 2> gpurun_out/benches_r02f/c0.err; echo c0=$?
python bench.py --config 1 --cpu-seconds 8 > gpurun_out/benches_r02f/c1.json 2> gpurun_out/benches_r02f/c1.err; echo c1=$?
for c in 3 2; do
  python bench.py --config $c --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/benches_r02f/c$c.json 2> gpurun_out/benches_r02f/c$c.err; echo c$c=$?
done
python bench.py --config 1 --dict dft --steps 20 --warmup 3 --cpu-seconds 8 > gpurun_out/benches_r02f/c1_dft.json 2> gpurun_out/benches_r02f/c1_dft.err; echo c1dft=$?
python bench.py --config 1 --dict union:dft+bdft --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/benches_r02f/c1_dftbdft.json 2> gpurun_out/benches_r02f/c1_dftbdft.err; echo c1dftbdft=$?
python bench.py --config 1 --recursion exact --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/benches_r02f/c1_exact.json 2> gpurun_out/benches_r02f/c1_exact.err; echo c1exact=$?
python bench.py --recursion exact --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/benches_r02f/c4_exact.json 2> gpurun_out/benches_r02f/c4_exact.err; echo c4exact=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/benches_r02f/c4_reference.json 2> gpurun_out/benches_r02f/c4_reference.err; echo ref=$?
for f in gpurun_out/benches_r02f/*.json; do echo "$f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d.get('e2e',{}).get('value',0)), d.get('clocks',{}).get('sm_mhz'), (d.get('parity_vs_reference') or {}).get('identical'))" 2>/dev/null)"; done
