# round 2, call AR: n = 8192 T0-T5 (W = 8) pass-1 group size
mkdir -p gpurun_out/r02ar
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02ar
for v in w8g4 w8g8 w8g2; do
  TT_LIB_PATH=variants/lib_$v.so TT_N=8192 TT_A=360 TT_REPS=3 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
done > $O/w8.txt 2>&1
cut -c1-150 $O/w8.txt
