set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -q -m "gpu and not slow" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 30 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -3 gpurun_out/bench.log
timeout 300 python bench.py --steps 30 --warmup 5 --sampler 1 --no-cpu-baseline > gpurun_out/bench_tex.log 2>&1; echo benchtex=$?
tail -3 gpurun_out/bench_tex.log
