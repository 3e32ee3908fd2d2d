# round 2, call CR: experiment -- TLD4 without the immediate texel offset (coordinate + 1 instead)
O=gpurun_out/r02cr
mkdir -p $O
run() { TT_LIB_PATH=$1 TT_N=$2 TT_A=$3 TT_FULL=1 TT_REPS=$4 timeout 180 python scripts/time_c2.py 2>&1 | tail -1 | sed "s#^#$1 #"; }
{
run variants/lib_cur.so 256 360 50; run variants/lib_na8.so 256 360 50
run variants/lib_cur.so 1024 720 20; run variants/lib_na32.so 1024 720 20
run variants/lib_cur.so 4096 1440 3; run variants/lib_na128.so 4096 1440 3
} > $O/ab.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02cr/ab.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],round(d['median_ms'],4), round(d['min_ms'],4), d['checksum'])
    except Exception: print(l[:300])
PY
