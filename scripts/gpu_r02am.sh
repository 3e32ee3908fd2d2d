# round 2, call AM: plan chunk cap for large images; plan tests + C3 bench
mkdir -p gpurun_out/r02am
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02am
timeout 900 python -m pytest tests/test_plan_gpu.py tests/test_batch_gpu.py -q -x > $O/pytest_plan.log 2>&1; echo pytest_plan=$?
tail -2 $O/pytest_plan.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
python -c "import json; d=json.load(open('$O/bench_c3.json')); print(d['ms_per_step'], d['e2e'])"
