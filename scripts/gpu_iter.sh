set -x
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -q -x -m "gpu" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -25 gpurun_out/pytest_gpu.log
python scripts/time_c2.py
TT_N=256 TT_A=360 python scripts/time_c2.py
TT_N=512 TT_A=360 python scripts/time_c2.py
TT_N=128 TT_A=360 python scripts/time_c2.py
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo benchc4=$?
python -c "import json; j=json.load(open('gpurun_out/bench_c4.json')); print('c4 ms', j['ms_per_step'], 'value %.3e'%j['value'], 'frac', j['roofline']['frac'])"
