# round 2, call CX: context sampler 3 (auto: TMA tiles for T0 launches of >= 1.5e8 taps): smoke, GPU suite, C5 sweep
O=gpurun_out/r02cx
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo PYTEST_EXIT $? >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 1500 python scripts/sweep.py > $O/sweep_c5.jsonl 2> $O/sweep_c5.err; echo sweep=$?
