# HBM regime: sweep of large n and one ncu capture of the 8192^2 T0-only (Radon) and T0-T5 launches
# (summaries exported on the box; the .ncu-rep files stay there: gpurun_out/ is capped at 64 MiB)
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
for f in 0 1; do
  tag=n8192_t0$([ $f = 1 ] && echo 5)
  TT_N=8192 TT_A=180 TT_FULL=$f TT_TAG=$tag bash scripts/prof_quick.sh
  python scripts/ncu_summary.py gpurun_out/prof_$tag.ncu-rep > gpurun_out/ncu_$tag.txt 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_${tag}_raw.csv 2>/dev/null
  rm -f gpurun_out/prof_$tag.ncu-rep
done
for cfg in "8192 360 0" "8192 360 1" "4096 1440 0" "4096 1440 1"; do
  set -- $cfg
  TT_N=$1 TT_A=$2 TT_FULL=$3 timeout 300 python scripts/time_c2.py
done
