# round 2, call BC: TMA Radon, two 64-line blocks per CTA -- parity, sanitizer, timings
mkdir -p gpurun_out/r02bc
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02bc
timeout 900 python -m pytest tests/test_radon_tma_gpu.py tests/test_parity_gpu.py tests/test_sharded_gpu.py tests/test_driver_gpu.py -q -x -k "tma or radon or non_finite or sampler or sharded" > $O/pytest.log 2>&1; echo pytest=$?
tail -2 $O/pytest.log
TT_N=2052 TT_A=6 timeout 300 compute-sanitizer --tool memcheck python scripts/tma_smoke.py > $O/memcheck.txt 2>&1; echo memcheck=$?; tail -2 $O/memcheck.txt
TT_N=1028 TT_A=5 timeout 300 compute-sanitizer --tool racecheck python scripts/tma_smoke.py > $O/racecheck.txt 2>&1; echo racecheck=$?; tail -2 $O/racecheck.txt
for cfg in "1024 720" "2048 720" "4096 1440" "8192 360" "16384 180"; do set -- $cfg
  TT_N=$1 TT_A=$2 TT_FULL=0 TT_SAMPLER_ID=2 TT_REPS=5 timeout 300 python scripts/time_c2.py 2>&1 | tail -1
done > $O/ab.txt 2>&1; cut -c1-130 $O/ab.txt
