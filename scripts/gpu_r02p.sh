# round 2, call P2: TMA Radon variants (taller boxes)
mkdir -p gpurun_out/r02p
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02p
for v in t32p0 t32p1 t32p2 t48p0 t48p1 t96p0 t96p1; do
  for cfg in "4096 1440" "8192 360"; do set -- $cfg
    TT_LIB_PATH=variants/lib_$v.so TT_N=$1 TT_A=$2 TT_FULL=0 TT_SAMPLER_ID=2 TT_REPS=5 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
  done
done > $O/tma_variants2.txt 2>&1
TT_N=4096 TT_A=1440 TT_FULL=0 TT_SAMPLER_ID=1 TT_REPS=5 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/tex /" >> $O/tma_variants2.txt
cat $O/tma_variants2.txt | cut -c1-150
