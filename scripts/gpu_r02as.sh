# round 2, call AS: sinogram-consumer stage timings; the paper's JIT-vs-native comparison on this build
mkdir -p gpurun_out/r02as
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02as
timeout 300 python scripts/time_pstages.py > $O/pstages.jsonl 2>&1; echo pstages=$?
cat $O/pstages.jsonl
timeout 900 python scripts/jit_vs_native.py > $O/jit_vs_native.jsonl 2>&1; echo jit=$?
cat $O/jit_vs_native.jsonl | cut -c1-300
