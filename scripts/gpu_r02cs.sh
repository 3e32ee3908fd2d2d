# round 2, call CS: final build -- smoke, GPU suite, bench C3 (default) + C1/C2, C3 launch list, ncu --set full of
# one C3 T0-T5 launch (profiles/ncu_c3_summary.json)
set -x
O=gpurun_out/r02cs; R=/tmp/r02cs; mkdir -p $O $R
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo bench_c3=$?
for w in c1 c2; do timeout 600 python bench.py --workload $w --steps 30 > $O/bench_$w.json 2> $O/bench_$w.err; echo bench_$w=$?; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launches_c3.log 2>&1; echo ncu_launches=$?
TT_N=4096 TT_A=1440 TT_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 -o $R/prof_c3 -f python scripts/time_c2.py > $O/prof_c3.log 2>&1; echo ncu_c3=$?
ncu -i $R/prof_c3.ncu-rep --page raw --csv > $O/ncu_c3_raw.csv 2>/dev/null
python scripts/ncu_summary.py $R/prof_c3.ncu-rep > $O/ncu_c3.txt 2>&1
