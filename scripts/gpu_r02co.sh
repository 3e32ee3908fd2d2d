# round 2, call CO: experiment -- TLD4 from a pitch-linear texture over the row-major image (no array copy) vs the
# block-linear cudaArray, C1 / C2 / C3 schedules
O=gpurun_out/r02co
mkdir -p $O
run() { TT_LIB_PATH=$1 TT_N=$2 TT_A=$3 TT_FULL=1 TT_REPS=$4 timeout 180 python scripts/time_c2.py 2>&1 | tail -1 | sed "s#^#$1 #"; }
{
run variants/lib_pk.so 256 360 50; run variants/lib_p8.so 256 360 50
run variants/lib_pk.so 1024 720 20; run variants/lib_p32.so 1024 720 20
run variants/lib_pk.so 4096 1440 3; run variants/lib_p128.so 4096 1440 3
} > $O/ab.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02co/ab.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],round(d['median_ms'],4), round(d['min_ms'],4), d['checksum'])
    except Exception: print(l[:300])
PY
