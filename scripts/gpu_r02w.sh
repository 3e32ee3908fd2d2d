# round 2, call W: C3 pass-1 pipelining / register-budget variants (W = 4 lines)
mkdir -p gpurun_out/r02w
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02w
for v in d128 g8 g8m2 g4m2 g6; do
  TT_LIB_PATH=variants/lib_$v.so TT_N=4096 TT_A=1440 TT_REPS=3 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
done > $O/c3_variants.txt 2>&1
cat $O/c3_variants.txt | cut -c1-200
