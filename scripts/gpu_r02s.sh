# round 2, call S: full GPU suite with the sampler-2 default (TMA Radon where eligible) + bench lines
mkdir -p gpurun_out/r02s
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02s
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo pytest_gpu=$?
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -2 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
cut -c1-400 $O/bench_c3.json
