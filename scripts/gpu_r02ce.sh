# round 2, call CE: gather assembly of ShardedTrace (tests + 2/4-rank one-GPU bench runs), the clipped-T0 parity test
mkdir -p gpurun_out/r02ce
O=gpurun_out/r02ce
python -m pytest tests/test_sharded_gpu.py "tests/test_parity_gpu.py::test_clipped_t0_off_grid_and_near_axis_angles" -q > $O/pytest.log 2>&1; echo PYTEST_EXIT $? >> $O/pytest.log
tail -3 $O/pytest.log
for g in 2 4; do
  timeout 600 python bench.py --gpus $g --workload c3 --dev-one-gpu --steps 5 --warmup 3 --no-cpu-baseline --assembly gather > $O/bench_c3_dev${g}_gather.json 2> $O/bench_c3_dev${g}_gather.err
  echo "dev$g gather rc=$?"; python -c "
import json; d=json.load(open('$O/bench_c3_dev${g}_gather.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d.get('e2e_matches_device_result'), d['config']['parallelism'])"
done
