# one ncu --set full capture of the fused kernel on C2 (or TT_N/TT_A), source-attributed
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
TT_SAMPLER_PROF=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 \
  -o gpurun_out/prof_${TT_TAG:-c2} -f python scripts/prof_c2.py > gpurun_out/prof_${TT_TAG:-c2}.log 2>&1; echo prof=$?
tail -2 gpurun_out/prof_${TT_TAG:-c2}.log
