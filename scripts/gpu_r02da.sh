# round 2, call DA: pitch-linear view vs array at n = 512 (NS = 16), T0-T5 and T0, kernel only
O=gpurun_out/r02da
mkdir -p $O
for full in 1 0; do for A in 360 1440; do for v in a512 v512; do
  TT_LIB_PATH=variants/lib_$v.so TT_N=512 TT_A=$A TT_FULL=$full TT_REPS=50 timeout 120 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
done; done; done > $O/ab.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02da/ab.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],d['full'],round(d['median_ms'],4), round(d['min_ms'],4), d['checksum'])
    except Exception: print(l[:200])
PY
