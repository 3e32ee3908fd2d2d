# round 2, call CC: tap-range clip with a reciprocal instead of divisions, C3 and C2 schedules
mkdir -p gpurun_out/r02cc
O=gpurun_out/r02cc
for v in c3_noclip c3_fast c3_fastp2 c3_noclip; do TT_LIB_PATH=variants/lib_$v.so TT_N=4096 TT_A=1440 TT_REPS=3 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"; done > $O/ab.txt 2>&1
for v in c2_noclip c2_fast c2_fastp2 c2_noclip; do TT_LIB_PATH=variants/lib_$v.so TT_N=1024 TT_A=720 TT_REPS=20 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"; done >> $O/ab.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02cc/ab.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],round(d['median_ms'],4), d['checksum'])
    except Exception: print(l[:150])
PY
