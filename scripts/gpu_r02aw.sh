# round 2, call AW: TMA vs texture Radon for 512 < n <= 1024 with 128-tap stages (threshold)
mkdir -p gpurun_out/r02aw
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02aw
for cfg in "516 360" "576 720" "640 720" "768 720" "896 720" "1024 720"; do set -- $cfg
  for smp in 1 2; do TT_LIB_PATH=variants/lib_m512.so TT_N=$1 TT_A=$2 TT_FULL=0 TT_SAMPLER_ID=$smp TT_REPS=20 TT_TEXPREP=1 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/smp=$smp /"; done
done > $O/thr.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02aw/thr.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],round(d['median_ms'],4))
    except Exception: print(l[:150])
PY
