# round 2, call CD: the adopted clip (T0 texture launches only): GPU suite + A/B against the previous build
mkdir -p gpurun_out/r02cd
O=gpurun_out/r02cd
cp paper_1604_03410_b200/libtt_b200.so variants/lib_new.so
for cfg in "256 360 0 50" "512 360 0 50" "640 720 0 20" "256 2880 0 20" "1024 720 1 20" "256 360 1 50"; do
  set -- $cfg
  for v in noclip new; do
    TT_LIB_PATH=variants/lib_$v.so TT_N=$1 TT_A=$2 TT_FULL=$3 TT_REPS=$4 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
  done
done > $O/ab.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02cd/ab.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],d['full'],round(d['median_ms'],5), d['checksum'])
    except Exception: print(l[:150])
PY
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo PYTEST_EXIT $? >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
