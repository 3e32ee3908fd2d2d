# round 2, call CN: compute-sanitizer over every kernel of the final build (TMA stage skipping, the new pitch
# kernel and the clipped texture T0 launches included), C5 sweep, GPU suite, smoke
O=gpurun_out/r02cn
mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 $O/sanitize_$tool.log
done
timeout 1500 python scripts/sweep.py > $O/sweep_c5.jsonl 2> $O/sweep_c5.err; echo sweep=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo PYTEST_EXIT $? >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
