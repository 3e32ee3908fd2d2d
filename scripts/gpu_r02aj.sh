# round 2, call AJ: TMA Radon with transposed tiles for near-vertical lines (on the current kernel)
mkdir -p gpurun_out/r02aj
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02aj
timeout 900 python -m pytest tests/test_radon_tma_gpu.py tests/test_parity_gpu.py -q -x -k "tma or radon or non_finite" > $O/pytest_tma.log 2>&1; echo pytest_tma=$?
tail -2 $O/pytest_tma.log
for v in tr0 tr1 tr1p2; do for cfg in "4096 1440" "8192 360" "2048 720" "1024 720"; do set -- $cfg
  TT_LIB_PATH=variants/lib_$v.so TT_N=$1 TT_A=$2 TT_FULL=0 TT_SAMPLER_ID=2 TT_REPS=5 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
done; done > $O/tr.txt 2>&1
cat $O/tr.txt | cut -c1-150
