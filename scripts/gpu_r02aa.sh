# round 2, call AA: C3 lines per CTA (W = 4): 2 (256 thr, 3 CTAs/SM), 3 (384, 2/SM), 6 (768, 1/SM)
mkdir -p gpurun_out/r02aa
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02aa
for v in b256 b384 b768; do
  TT_LIB_PATH=variants/lib_$v.so TT_N=4096 TT_A=1440 TT_REPS=3 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
done > $O/c3_cta.txt 2>&1
cat $O/c3_cta.txt | cut -c1-200
