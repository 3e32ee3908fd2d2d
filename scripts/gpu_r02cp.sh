# round 2, call CP: pitch-linear texture views for n <= 256 (no array copy): GPU suite, smoke, C1 bench
O=gpurun_out/r02cp
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo PYTEST_EXIT $? >> $O/pytest_gpu.log; tail -4 $O/pytest_gpu.log
timeout 600 python bench.py --workload c1 --steps 50 > $O/bench_c1.json 2> $O/bench_c1.err; echo bench_c1=$?
python -c "
import json; d=json.load(open('$O/bench_c1.json')); print(d['ms_per_step'], d['value'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['roofline'].get('kernel_ms'))"
