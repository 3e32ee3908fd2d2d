# round 2, call CV: T0 crossover texture (clipped) vs TMA tiles (stage skipping off below 2048, parallel pitch kernel)
O=gpurun_out/r02cv
mkdir -p $O
for cfg in "704 360" "704 1440" "768 360" "768 1440" "896 720" "1024 180" "1024 720" "1024 2880"; do
  set -- $cfg
  for smp in 1 2; do
    TT_SAMPLER_ID=$smp TT_N=$1 TT_A=$2 TT_FULL=0 TT_REPS=30 timeout 120 python scripts/time_c2.py 2>&1 | tail -1
  done
done > $O/ab.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02cv/ab.txt'):
    try: d=json.loads(l); print(d['n'],d['A'],d['sampler'],round(d['median_ms'],4), d['checksum'])
    except Exception: print(l[:200])
PY
