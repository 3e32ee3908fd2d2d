set -x
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 -o gpurun_out/prof_c2_ldg -f python scripts/prof_c2.py > gpurun_out/prof_ldg.log 2>&1; echo ldg=$?
TT_SAMPLER_PROF=1 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 -o gpurun_out/prof_c2_tex -f python scripts/prof_c2.py > gpurun_out/prof_tex.log 2>&1; echo tex=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; echo launches=$?
ls -la gpurun_out
