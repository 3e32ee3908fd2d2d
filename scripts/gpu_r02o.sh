# round 2, call O: TMA probe -- box x alignment vs cluster launch
mkdir -p gpurun_out/r02o
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tpp scripts/probes/tma_param_probe.cu -lcuda
( echo "== plain launch x=12"; timeout 60 /tmp/tpp 0 64 12 1 0 0;
  echo "== plain launch x=-4"; timeout 60 /tmp/tpp 0 64 -4 1 0 0;
  echo "== plain launch x=12 global map"; timeout 60 /tmp/tpp 2 64 12 1 0 0;
  echo "== plain launch x=12 array map"; timeout 60 /tmp/tpp 1 128 12 1 0 0;
  echo "== cluster launch x=10"; timeout 60 /tmp/tpp 0 64 10 1 0 1 ) > $O/tma_param_probe4.txt 2>&1
cat $O/tma_param_probe4.txt | grep -v "desc\|entry"
