# round 2, call L: P stage separate by default (fused opt-in); full GPU suite + C1/C2/C3 bench lines
mkdir -p gpurun_out/r02l
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02l
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo pytest_gpu=$?
tail -3 $O/pytest_gpu.log
for cfg in "1024 720" "256 360" "2048 720"; do set -- $cfg
  for c in 0 1 2; do TT_N=$1 TT_A=$2 TT_CIRC=$c TT_REPS=20 timeout 300 python scripts/time_c2.py | sed "s/^/circ=$c /"; done
done > $O/time_circ.txt 2>&1
cat $O/time_circ.txt | cut -c1-140
timeout 600 python bench.py --workload c2 --steps 30 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err; echo c2=$?
timeout 600 python bench.py --workload c1 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err; echo c1=$?
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02l/bench_*.json')):
    try:
        d=json.load(open(f)); r=d['roofline']
        print(f, d['ms_per_step'], d['e2e'].get('ms_per_step'), r.get('kernel_ms'), round(r['frac'],3), d['clocks'], d.get('gpu_launches'))
    except Exception as e: print(f, 'ERR', e)
PY
