# quick GPU check: parity tests + bench summary line
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'], 'iter_frac', round(d['roofline']['frac'],3), 'init_tf', round(d['roofline_init']['achieved'],2), 'gram_tf', round(d['gram_tflops'],2), 'e2e', d['e2e']['value'])"
