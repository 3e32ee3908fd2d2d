# round 2, call U: TMA Radon with transposed tiles for near-vertical lines
mkdir -p gpurun_out/r02u
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02u
timeout 900 python -m pytest tests/test_radon_tma_gpu.py -q -x > $O/pytest_tma.log 2>&1; echo pytest_tma=$?
tail -3 $O/pytest_tma.log
for cfg in "2048 720" "4096 1440" "8192 360" "3000 720" "16384 180" "8192 2880"; do set -- $cfg
  for smp in 1 2; do TT_N=$1 TT_A=$2 TT_FULL=0 TT_SAMPLER_ID=$smp TT_REPS=5 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/smp=$smp /"; done
done > $O/ab_t0.txt 2>&1
cat $O/ab_t0.txt | cut -c1-150
R=/tmp/r02u; mkdir -p $R
TT_N=4096 TT_A=1440 TT_FULL=0 TT_SAMPLER_ID=2 TT_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:radon_tma -s 1 -c 1 -o $R/prof_t0_tma -f python scripts/time_c2.py > $O/prof_t0_tma.log 2>&1; echo ncu_tma=$?
TT_N=4096 TT_A=1440 TT_FULL=0 TT_SAMPLER_ID=1 TT_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 -o $R/prof_t0_tex -f python scripts/time_c2.py > $O/prof_t0_tex.log 2>&1; echo ncu_tex=$?
for k in tma tex; do
  python scripts/ncu_summary.py $R/prof_t0_$k.ncu-rep > $O/ncu_t0_$k.txt 2>&1
  ncu -i $R/prof_t0_$k.ncu-rep --page raw --csv > $O/ncu_t0_${k}_raw.csv 2>/dev/null
  ncu -i $R/prof_t0_$k.ncu-rep --page source --csv --print-source sass > $O/ncu_t0_${k}_sass.csv 2>/dev/null
done
head -32 $O/ncu_t0_tma.txt
ls -la $O
