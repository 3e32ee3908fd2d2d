# iteration: tests, bench variants, ncu of the C2 kernel
set -x
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -q -x -m "gpu and not slow" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
for smp in 1 0; do
  timeout 300 python bench.py --steps 30 --warmup 5 --sampler $smp --no-cpu-baseline > gpurun_out/bench_s$smp.log 2>&1; echo bench=$?
  tail -1 gpurun_out/bench_s$smp.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c2 sampler', $smp, 'ms', round(j['ms_per_step'],4), 'value %.3e'%j['value'], 'frac', round(j['roofline']['frac'],4), 'e2e %.3e'%j['e2e']['value'])"
done
TT_SAMPLER_PROF=1 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 -o gpurun_out/prof_c2_s1 -f python scripts/prof_c2.py > gpurun_out/prof_s1.log 2>&1; echo prof=$?
