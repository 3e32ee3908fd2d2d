# round 2, call A: GPU tests, line-block visiting order A/B at large n, ncu of C3 and 8192^2
mkdir -p gpurun_out/r02a
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02a
timeout 1200 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 $O/pytest_gpu.log
for pb in 0 64 128 256 512 1024; do
  for cfg in "4096 1440 1" "8192 360 1" "8192 360 0" "2048 720 1"; do
    set -- $cfg
    TT_PBLOCK=$pb TT_N=$1 TT_A=$2 TT_FULL=$3 TT_REPS=6 timeout 300 python scripts/time_c2.py | sed "s/^/pb=$pb /"
  done
done > $O/pblock.txt 2>&1
cat $O/pblock.txt
for pb in 0 256; do
  for cfg in "4096 1440 1 c3" "8192 180 1 n8192_t05" "8192 180 0 n8192_t0"; do
    set -- $cfg
    TT_PBLOCK=$pb TT_N=$1 TT_A=$2 TT_FULL=$3 TT_REPS=1 TT_SAMPLER_PROF=1 timeout 600 ncu --set full --clock-control none \
      --import-source on -k regex:trace_kernel -s 0 -c 1 -o $O/prof_${4}_pb$pb -f python scripts/prof_c2.py > $O/prof_${4}_pb$pb.log 2>&1
    python scripts/ncu_summary.py $O/prof_${4}_pb$pb.ncu-rep > $O/ncu_${4}_pb$pb.txt 2>&1
    ncu -i $O/prof_${4}_pb$pb.ncu-rep --page raw --csv > $O/ncu_${4}_pb${pb}_raw.csv 2>/dev/null
  done
done
rm -f $O/prof_n8192*.ncu-rep
ls -la $O
