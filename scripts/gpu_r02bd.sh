# round 2, call BD: persistent T0-T5 grid (resident CTAs striding over the lines) vs one CTA per line group
mkdir -p gpurun_out/r02bd
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02bd
for v in c3p0 c3p1; do TT_LIB_PATH=variants/lib_$v.so TT_N=4096 TT_A=1440 TT_REPS=3 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"; done > $O/persist.txt 2>&1
for v in c2p0 c2p1; do TT_LIB_PATH=variants/lib_$v.so TT_N=1024 TT_A=720 TT_REPS=20 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"; done >> $O/persist.txt 2>&1
for v in c1p0 c1p1; do TT_LIB_PATH=variants/lib_$v.so TT_N=256 TT_A=360 TT_REPS=50 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"; done >> $O/persist.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02bd/persist.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],round(d['median_ms'],4), d['checksum'])
    except Exception: print(l[:150])
PY
