# round 2, call CK: TMA map cache (host encode once per image address) A/B at short T0 launches
O=gpurun_out/r02ck
mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
for cfg in "1024 180" "1024 360" "2048 180" "1024 720" "4096 1440"; do
  set -- $cfg
  for v in tpl mapc; do
    TT_SAMPLER_ID=2 TT_LIB_PATH=variants/lib_$v.so TT_N=$1 TT_A=$2 TT_FULL=0 TT_REPS=30 timeout 120 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
  done
done > $O/ab.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02ck/ab.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],d['sampler'],round(d['median_ms'],4), round(d['min_ms'],4), d['checksum'])
    except Exception: print(l[:200])
PY
TT_SAMPLER_ID=2 TT_LIB_PATH=variants/lib_mapc.so TT_N=1024 TT_A=180 TT_FULL=0 TT_REPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/time_c2.py 2>/dev/null | grep -i "radon\|pitch" | awk -F'","' '{print $5, $NF}' | cut -c1-60,200- | tail -6
