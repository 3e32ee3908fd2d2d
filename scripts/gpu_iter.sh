mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m "gpu" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for cfg in "1024 720" "256 360" "4096 90"; do set -- $cfg; TT_N=$1 TT_A=$2 python scripts/time_c2.py; done
