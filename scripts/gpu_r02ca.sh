# round 2, call CA: clipped tap range (TT_CLIP) A/B vs the unclipped build, then the GPU suite on the clipped build
mkdir -p gpurun_out/r02ca
O=gpurun_out/r02ca
for cfg in "256 360 1 50" "1024 720 1 20" "4096 1440 1 3" "2048 720 1 5" "1000 720 1 10" "512 360 0 50" "8192 180 1 2"; do
  set -- $cfg
  for v in noclip clip; do
    TT_LIB_PATH=variants/lib_$v.so TT_N=$1 TT_A=$2 TT_FULL=$3 TT_REPS=$4 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"
  done
done > $O/clip_ab.txt 2>&1
cat $O/clip_ab.txt
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo PYTEST_EXIT $? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
