# round 2, call CF: TMA Radon stage skipping (tiles that miss the image): parity + A/B vs the previous build
mkdir -p gpurun_out/r02cf
O=gpurun_out/r02cf
cp paper_1604_03410_b200/libtt_b200.so variants/lib_skip.so
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo PYTEST_EXIT $? >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
for cfg in "1024 720 20" "2048 720 10" "4096 1440 5" "8192 360 3" "16384 180 3"; do
  set -- $cfg
  for v in noclip skip; do
    TT_SAMPLER_ID=2 TT_LIB_PATH=variants/lib_$v.so TT_N=$1 TT_A=$2 TT_FULL=0 TT_REPS=$3 timeout 120 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
  done
done > $O/ab.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02cf/ab.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],d['sampler'],round(d['median_ms'],4), d['checksum'])
    except Exception: print(l[:200])
PY
