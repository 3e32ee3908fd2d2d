# round 2, call AP: pass-1 groups of 8 taps for sub-warp T0-T5 segments (n <= 512): parity + timings + C4/C1 bench
mkdir -p gpurun_out/r02ap
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02ap
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_batch_gpu.py tests/test_reference_configs_gpu.py -q -x > $O/pytest.log 2>&1; echo pytest=$?
tail -2 $O/pytest.log
for cfg in "128 360" "256 360" "512 360" "256 720" "384 360"; do set -- $cfg
  TT_N=$1 TT_A=$2 TT_REPS=50 timeout 300 python scripts/time_c2.py 2>&1 | tail -1
done > $O/small.txt 2>&1
cut -c1-130 $O/small.txt
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo c4=$?
timeout 600 python bench.py --workload c1 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err; echo c1=$?
python -c "
import json
for w in ('c1','c4'):
    d=json.load(open('$O/bench_'+w+'.json')); print(w, d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'])"
