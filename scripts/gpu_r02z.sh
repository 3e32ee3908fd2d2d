# round 2, call Z: TMA Radon, tail stage split out
mkdir -p gpurun_out/r02z
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02z
timeout 900 python -m pytest tests/test_radon_tma_gpu.py -q -x > $O/pytest_tma.log 2>&1; echo pytest_tma=$?
tail -2 $O/pytest_tma.log
for cfg in "2048 720" "4096 1440" "8192 360" "16384 180"; do set -- $cfg
  TT_N=$1 TT_A=$2 TT_FULL=0 TT_SAMPLER_ID=2 TT_REPS=5 timeout 300 python scripts/time_c2.py 2>&1 | tail -1
done > $O/ab_t0.txt 2>&1
cat $O/ab_t0.txt | cut -c1-130
