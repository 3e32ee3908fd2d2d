set -x
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -q -x -m "gpu" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
cat gpurun_out/bench_c2.json; tail -3 gpurun_out/bench_c2.err
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo benchc4=$?
cat gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
