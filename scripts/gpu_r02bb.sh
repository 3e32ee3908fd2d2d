# round 2, call BB: TMA Radon line blocks per CTA (ring continues across blocks)
mkdir -p gpurun_out/r02bb
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02bb
for v in b1 b2; do for cfg in "4096 1440" "8192 360" "2048 720" "1024 720" "3000 720"; do set -- $cfg
  TT_LIB_PATH=variants/lib_$v.so TT_N=$1 TT_A=$2 TT_FULL=0 TT_SAMPLER_ID=2 TT_REPS=5 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
done; done > $O/blocks.txt 2>&1
TT_LIB_PATH=variants/lib_b1.so TT_N=3000 TT_A=720 TT_FULL=0 TT_SAMPLER_ID=1 TT_REPS=2 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/tex /" >> $O/blocks.txt
python - <<'PY'
import json
for l in open('gpurun_out/r02bb/blocks.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],round(d['median_ms'],3), d['checksum'])
    except Exception: print(l[:150])
PY
