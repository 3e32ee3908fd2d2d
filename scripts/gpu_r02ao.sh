# round 2, call AO: C1 (n = 256, LG = 8 segments) pass-1 group size and register budget
mkdir -p gpurun_out/r02ao
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02ao
for v in s8 s8g8 s8m13 s8m16; do
  TT_LIB_PATH=variants/lib_$v.so TT_N=256 TT_A=360 TT_REPS=50 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
done > $O/c1_variants.txt 2>&1
cut -c1-150 $O/c1_variants.txt
