# full evidence run: all GPU tests, smoke, bench (+reference arm), ncu launch list + full capture, C5 sweep
set -x
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
nproc; lscpu | grep "Model name"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; cat gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo benchref=$?
cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; echo launches=$?
TT_SAMPLER_PROF=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 -o gpurun_out/prof_c2 -f python scripts/prof_c2.py > gpurun_out/prof_c2.log 2>&1; echo prof=$?
timeout 600 ncu --set full --clock-control none -k regex:circus_kernel -s 1 -c 1 -o gpurun_out/prof_circus -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof_circus.log 2>&1; echo profcircus=$?
timeout 900 python scripts/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo sweep=$?
tail -3 gpurun_out/sweep.jsonl
