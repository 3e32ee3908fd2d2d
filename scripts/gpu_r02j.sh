# round 2, call J: fused-P-stage cost breakdown (TT_EPI_MODE variants) + shared-memory sampling probe
mkdir -p gpurun_out/r02j
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02j
for m in 0 1 2 3; do
  for c in 0 1; do
    TT_LIB_PATH=variants/lib_e8_$m.so TT_N=256 TT_A=360 TT_CIRC=$c TT_REPS=20 timeout 120 python scripts/time_c2.py | sed "s/^/e8 mode=$m circ=$c /"
    TT_LIB_PATH=variants/lib_e32_$m.so TT_N=1024 TT_A=720 TT_CIRC=$c TT_REPS=20 timeout 120 python scripts/time_c2.py | sed "s/^/e32 mode=$m circ=$c /"
  done
done > $O/epi_modes.txt 2>&1
cat $O/epi_modes.txt | cut -c1-150
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ssp scripts/probes/smem_sample_probe.cu && /tmp/ssp > $O/smem_sample_probe.json 2>&1
cat $O/smem_sample_probe.json
