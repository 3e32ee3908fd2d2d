# round 2, call CH: adaptive blocks per CTA for the TMA Radon kernel; small-n texture T0 clip check
O=gpurun_out/r02ch
mkdir -p $O
for cfg in "1024 180 2" "1024 360 2" "2048 180 2" "1024 720 2" "4096 1440 2" "256 180 1" "256 360 1" "128 360 1"; do
  set -- $cfg
  for v in noclip skip bpc; do
    TT_SAMPLER_ID=$3 TT_LIB_PATH=variants/lib_$v.so TT_N=$1 TT_A=$2 TT_FULL=0 TT_REPS=50 timeout 120 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
  done
done > $O/ab.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02ch/ab.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],d['sampler'],round(d['median_ms'],4), round(d['min_ms'],4), d['checksum'])
    except Exception: print(l[:200])
PY
timeout 600 python -m pytest tests/test_radon_tma_gpu.py tests/test_parity_gpu.py -x -q > $O/pytest.log 2>&1; echo PYTEST_EXIT $? >> $O/pytest.log; tail -2 $O/pytest.log
