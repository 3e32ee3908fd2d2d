# round 2, call K: raw-entry scratch pool kept; fused vs separate P stage
mkdir -p gpurun_out/r02k
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02k
timeout 900 python -m pytest tests/test_circus_gpu.py tests/test_plan_gpu.py tests/test_batch_gpu.py tests/test_parity_gpu.py -q -x > $O/pytest_a.log 2>&1; echo pytest_a=$?
tail -3 $O/pytest_a.log
for cfg in "1024 720" "256 360" "512 360" "2048 720"; do set -- $cfg
  for c in 0 1; do TT_N=$1 TT_A=$2 TT_CIRC=$c TT_REPS=20 timeout 300 python scripts/time_c2.py | sed "s/^/circ=$c /"; done
done > $O/time_circ.txt 2>&1
cat $O/time_circ.txt
TT_N=4096 TT_A=1440 TT_REPS=3 timeout 300 python scripts/time_c2.py > $O/time_c3.txt 2>&1; cat $O/time_c3.txt
for f in 0 1; do
  TT_FUSED_CIRCUS=$f timeout 600 python bench.py --workload c2 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_c2_fused$f.json 2> $O/bench_c2_fused$f.err; echo c2_fused$f=$?
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
TT_CIRC=1 TT_REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_fused.csv python scripts/time_c2.py > /dev/null 2>&1; echo ncu=$?
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02k/bench_*.json')):
    try:
        d=json.load(open(f)); r=d['roofline']
        print(f, d['ms_per_step'], d['e2e'].get('ms_per_step'), r.get('kernel_ms'), round(r['frac'],3), d['clocks'])
    except Exception as e: print(f, 'ERR', e)
PY
