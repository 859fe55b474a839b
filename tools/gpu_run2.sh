cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/i8_peak_probe tools/probes/i8_peak_probe.cu && timeout 60 gpurun_out/i8_peak_probe > gpurun_out/i8_peak.json; echo i8=$?; cat gpurun_out/i8_peak.json
timeout 600 python bench.py > gpurun_out/b4_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/b4_default.log | cut -c1-3000
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref4.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/ref4.log | cut -c1-600
timeout 300 python bench.py --config 1 --steps 20 --no-cpu-baseline > gpurun_out/b1.log 2>&1; echo "c1 rc=$?"; tail -1 gpurun_out/b1.log | cut -c1-400
timeout 300 python bench.py --config 3 --steps 10 --no-cpu-baseline > gpurun_out/b3.log 2>&1; echo "c3 rc=$?"; tail -1 gpurun_out/b3.log | cut -c1-400
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_all.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_all.log
