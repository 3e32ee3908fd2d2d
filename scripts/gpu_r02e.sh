# round 2, call E: fused P stage v2 (CTA counting, grid-tail drainers), graphs per slot stream, f4 kernels
mkdir -p gpurun_out/r02e
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02e
timeout 900 python -m pytest tests/test_circus_gpu.py tests/test_plan_gpu.py tests/test_functionals_f4_gpu.py -q -x > $O/pytest_a.log 2>&1; echo pytest_a=$?
tail -15 $O/pytest_a.log
for f in 0 1; do
  TT_FUSED_CIRCUS=$f timeout 600 python bench.py --workload c2 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_c2_fused$f.json 2> $O/bench_c2_fused$f.err; echo c2_fused$f=$?
done
timeout 600 python bench.py --workload c1 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err; echo c1=$?
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo c4=$?
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo pytest_gpu=$?
tail -3 $O/pytest_gpu.log
ls -la $O
