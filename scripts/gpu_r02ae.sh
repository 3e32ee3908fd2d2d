# round 2, call AE: TMA Radon with a zero footprint for out-of-range taps
mkdir -p gpurun_out/r02ae
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02ae
timeout 900 python -m pytest tests/test_radon_tma_gpu.py -q -x > $O/pytest_tma.log 2>&1; echo pytest_tma=$?
tail -2 $O/pytest_tma.log
for cfg in "516 360" "768 360" "1000 720" "1024 720" "1024 2880" "2048 720" "4096 1440" "8192 360"; do set -- $cfg
  for smp in 2; do TT_N=$1 TT_A=$2 TT_FULL=0 TT_SAMPLER_ID=$smp TT_REPS=10 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/smp=$smp /"; done
done > $O/ab_t0.txt 2>&1
cat $O/ab_t0.txt | cut -c1-130
