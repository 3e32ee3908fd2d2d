# round 2, call C: fused P stage parity + full GPU suite; C2 fused vs separate circus; C3 bench with traffic
mkdir -p gpurun_out/r02c
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02c
timeout 600 python -m pytest tests/test_circus_gpu.py tests/test_plan_gpu.py -q -x > $O/pytest_circus.log 2>&1; echo pytest_circus=$?
tail -3 $O/pytest_circus.log
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo pytest_gpu=$?
tail -3 $O/pytest_gpu.log
for f in 0 1; do
  TT_FUSED_CIRCUS=$f timeout 600 python bench.py --workload c2 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_c2_fused$f.json 2> $O/bench_c2_fused$f.err; echo c2_fused$f=$?
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_c2_bench.log 2>&1
ls -la $O
