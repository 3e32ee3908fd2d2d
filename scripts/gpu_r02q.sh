# round 2, call Q: TMA Radon default build (one 96-row box per stage) -- parity, A/B sweep, ncu, stage variants
mkdir -p gpurun_out/r02q
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02q
timeout 900 python -m pytest tests/test_radon_tma_gpu.py tests/test_parity_gpu.py -q -x -k "tma or radon" > $O/pytest_tma.log 2>&1; echo pytest_tma=$?
tail -3 $O/pytest_tma.log
for cfg in "2048 720" "4096 1440" "8192 360" "3000 720" "16384 180" "8192 2880"; do set -- $cfg
  for smp in 1 2; do TT_N=$1 TT_A=$2 TT_FULL=0 TT_SAMPLER_ID=$smp TT_REPS=5 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/smp=$smp /"; done
done > $O/ab_t0.txt 2>&1
for v in s3 s5; do TT_LIB_PATH=variants/lib_$v.so TT_N=4096 TT_A=1440 TT_FULL=0 TT_SAMPLER_ID=2 TT_REPS=5 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"; done >> $O/ab_t0.txt
cat $O/ab_t0.txt | cut -c1-150
TT_N=4096 TT_A=1440 TT_FULL=0 TT_SAMPLER_ID=2 TT_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:radon_tma -s 1 -c 1 -o $O/prof_t0_tma -f python scripts/time_c2.py > $O/prof_t0_tma.log 2>&1; echo ncu_tma=$?
TT_N=4096 TT_A=1440 TT_FULL=0 TT_SAMPLER_ID=1 TT_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 -o $O/prof_t0_tex -f python scripts/time_c2.py > $O/prof_t0_tex.log 2>&1; echo ncu_tex=$?
python scripts/ncu_summary.py $O/prof_t0_tma.ncu-rep > $O/ncu_t0_tma.txt 2>&1
python scripts/ncu_summary.py $O/prof_t0_tex.ncu-rep > $O/ncu_t0_tex.txt 2>&1
head -30 $O/ncu_t0_tma.txt
