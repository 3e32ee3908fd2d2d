# round 2, call CI: stage skipping as its own instantiation (n >= 2048), T0 clip only for NS >= 16: A/B + GPU suite
O=gpurun_out/r02ci
mkdir -p $O
for cfg in "1024 720 2" "1024 360 2" "2048 720 2" "4096 1440 2" "8192 360 2" "256 360 1" "128 360 1" "512 360 1" "640 720 1"; do
  set -- $cfg
  for v in noclip tpl; do
    TT_SAMPLER_ID=$3 TT_LIB_PATH=variants/lib_$v.so TT_N=$1 TT_A=$2 TT_FULL=0 TT_REPS=30 timeout 120 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
  done
done > $O/ab.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02ci/ab.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],d['sampler'],round(d['median_ms'],4), round(d['min_ms'],4), d['checksum'])
    except Exception: print(l[:200])
PY
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo PYTEST_EXIT $? >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
