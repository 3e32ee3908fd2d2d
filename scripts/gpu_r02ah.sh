# round 2, call AH: TMA Radon stage-loop unroll
mkdir -p gpurun_out/r02ai
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02ai
for v in u1 u2 u4; do for cfg in "4096 1440" "8192 360" "2048 720"; do set -- $cfg
  TT_LIB_PATH=variants/lib_$v.so TT_N=$1 TT_A=$2 TT_FULL=0 TT_SAMPLER_ID=2 TT_REPS=5 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
done; done > $O/unroll.txt 2>&1
cat $O/unroll.txt | cut -c1-150
