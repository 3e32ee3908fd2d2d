# quick GPU check: parity tests + kernel timings (C2, C1-size, C3-size) + default bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
for cfg in "1024 720" "256 360" "512 360" "2048 720" "4096 1440"; do
  set -- $cfg
  TT_N=$1 TT_A=$2 timeout 300 python scripts/time_c2.py
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo bench=$?
cat gpurun_out/bench_quick.json
