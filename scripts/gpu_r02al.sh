# round 2, call AL: pass-2 unroll at C3 (W = 4) and C2 (W = 1)
mkdir -p gpurun_out/r02al
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02al
for v in u1 u2 u3 u4; do
  TT_LIB_PATH=variants/lib_$v.so TT_N=4096 TT_A=1440 TT_REPS=3 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
done > $O/p2unroll.txt 2>&1
for v in c2u2 c2u3; do
  TT_LIB_PATH=variants/lib_$v.so TT_N=1024 TT_A=720 TT_REPS=20 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
done >> $O/p2unroll.txt 2>&1
cut -c1-150 $O/p2unroll.txt
