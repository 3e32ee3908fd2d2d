# round 2, call AZ: TMA Radon pitch candidates with 128-tap stages
mkdir -p gpurun_out/r02az
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02az
for v in q2k1 q8k1 q8k2 q8k3; do for cfg in "4096 1440" "8192 360" "2048 720"; do set -- $cfg
  TT_LIB_PATH=variants/lib_$v.so TT_N=$1 TT_A=$2 TT_FULL=0 TT_SAMPLER_ID=2 TT_REPS=5 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
done; done > $O/padk.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02az/padk.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],round(d['median_ms'],3))
    except Exception: print(l[:150])
PY
