# iteration: tests, bench variants (sampler x warps-per-line), ncu of the C2 kernel
set -x
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -q -x -m "gpu and not slow" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
for W in 1 2; do for smp in 0 1; do
  TT_WARPS_PER_LINE=$W timeout 300 python bench.py --steps 30 --warmup 5 --sampler $smp --no-cpu-baseline > gpurun_out/bench_w${W}_s$smp.log 2>&1; echo bench=$?
  tail -1 gpurun_out/bench_w${W}_s$smp.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('W', $W, 'sampler', $smp, 'ms', round(j['ms_per_step'],4), 'value %.3e'%j['value'], 'frac', round(j['roofline']['frac'],4), 'e2e %.3e'%j['e2e']['value'])"
done; done
for W in 1 2; do
  TT_WARPS_PER_LINE=$W TT_SAMPLER_PROF=1 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 -o gpurun_out/prof_c2_w${W}_s1 -f python scripts/prof_c2.py > gpurun_out/prof_w${W}.log 2>&1; echo prof=$?
done
