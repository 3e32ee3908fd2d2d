# round 2, call CM: the pitch-selection kernel with one warp per (candidate, sample): A/B + TMA tests
O=gpurun_out/r02cm
mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
for cfg in "1024 180" "1024 360" "2048 180" "1024 720" "2048 720" "4096 1440" "8192 360"; do
  set -- $cfg
  for v in mapc pk; do
    TT_SAMPLER_ID=2 TT_LIB_PATH=variants/lib_$v.so TT_N=$1 TT_A=$2 TT_FULL=0 TT_REPS=30 timeout 120 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
  done
done > $O/ab.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02cm/ab.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],d['sampler'],round(d['median_ms'],4), round(d['min_ms'],4), d['checksum'])
    except Exception: print(l[:200])
PY
TT_SAMPLER_ID=2 TT_N=1024 TT_A=180 TT_FULL=0 TT_REPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/time_c2.py > $O/ncu_1024_180.csv 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r02cm/ncu_1024_180.csv')) if len(r)>10 and r[0]!='ID']
for r in rows[:6]: print(r[4][:40], r[12], r[14])
PY
timeout 600 python -m pytest tests/test_radon_tma_gpu.py -q > $O/pytest.log 2>&1; echo PYTEST_EXIT $? >> $O/pytest.log; tail -2 $O/pytest.log
