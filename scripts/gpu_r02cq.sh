# round 2, call CQ: texture-handle test, bench C1/C2 of the pitch-view build
O=gpurun_out/r02cq
mkdir -p $O
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "texture" > $O/pytest.log 2>&1; echo PYTEST_EXIT $? >> $O/pytest.log; tail -2 $O/pytest.log
for w in c1 c2; do timeout 600 python bench.py --workload $w --steps 30 > $O/bench_$w.json 2> $O/bench_$w.err; echo bench_$w=$?; done
