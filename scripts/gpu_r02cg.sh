# round 2, call CG: evidence of this build (smoke, GPU suite, bench C1-C4, C5 sweep, C3 launch list,
# ncu --set full of the TMA Radon kernel with stage skipping)
set -x
O=gpurun_out/r02cg
mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo bench_c3=$?
for w in c1 c2 c4; do timeout 600 python bench.py --workload $w --steps 20 > $O/bench_$w.json 2> $O/bench_$w.err; echo bench_$w=$?; done
timeout 1500 python scripts/sweep.py > $O/sweep_c5.jsonl 2> $O/sweep_c5.err; echo sweep=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launches_c3.log 2>&1; echo ncu_launches=$?
TT_N=4096 TT_A=1440 TT_FULL=0 TT_SAMPLER_ID=2 TT_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:radon_tma -s 1 -c 1 -o $O/prof_t0_tma -f python scripts/time_c2.py > $O/prof_t0_tma.log 2>&1; echo ncu_tma=$?
ncu -i $O/prof_t0_tma.ncu-rep --page raw --csv > $O/ncu_t0_tma_raw.csv 2>/dev/null
rm -f $O/prof_t0_tma.ncu-rep
