# round 2, call X: GPU suite (non-finite pixel parity, IpcBuffer) + 2/4-rank sharded C3 on one GPU
mkdir -p gpurun_out/r02x
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02x
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo pytest_gpu=$?
tail -3 $O/pytest_gpu.log
for g in 2 4; do
  timeout 900 python bench.py --gpus $g --workload c3 --dev-one-gpu --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3_dev$g.json 2> $O/bench_c3_dev$g.err; echo dev$g=$?
  python -c "import json; d=json.load(open('$O/bench_c3_dev$g.json')); print($g, d['ms_per_step'], d['e2e']['ms_per_step'], {k:v for k,v in d.items() if 'match' in k})"
done
