# round 2, call G (fresh container): full GPU suite on the restored last commit + C1/C2/C3 bench lines
mkdir -p gpurun_out/r02g
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02g
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 600 > $O/pytest_gpu.log 2>&1; echo pytest_gpu=$?
tail -15 $O/pytest_gpu.log
for f in 0 1; do
  TT_FUSED_CIRCUS=$f timeout 600 python bench.py --workload c2 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_c2_fused$f.json 2> $O/bench_c2_fused$f.err; echo c2_fused$f=$?
done
timeout 600 python bench.py --workload c1 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err; echo c1=$?
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err; echo default=$?
cat $O/bench_*.json | cut -c1-600
ls -la $O
