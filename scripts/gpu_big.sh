# HBM regime: sweep of large n and one ncu capture of the 8192^2 T0-only (Radon) launch
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
TT_N=8192 TT_A=180 TT_FULL=0 TT_TAG=n8192_t0 bash scripts/prof_quick.sh
TT_N=8192 TT_A=180 TT_FULL=1 TT_TAG=n8192_t05 bash scripts/prof_quick.sh
for cfg in "8192 360 0" "8192 360 1" "4096 1440 0" "4096 1440 1"; do
  set -- $cfg
  TT_N=$1 TT_A=$2 TT_FULL=$3 timeout 300 python scripts/time_c2.py
done
