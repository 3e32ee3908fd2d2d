# round 2, call AY: ncu of the 128-tap-stage TMA Radon kernel
mkdir -p gpurun_out/r02ay
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02ay; R=/tmp/r02ay; mkdir -p $R
TT_N=4096 TT_A=1440 TT_FULL=0 TT_SAMPLER_ID=2 TT_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:radon_tma -s 1 -c 1 -o $R/prof_t0_tma -f python scripts/time_c2.py > $O/prof_t0_tma.log 2>&1; echo ncu_tma=$?
python scripts/ncu_summary.py $R/prof_t0_tma.ncu-rep > $O/ncu_t0_tma.txt 2>&1
ncu -i $R/prof_t0_tma.ncu-rep --page raw --csv > $O/ncu_t0_tma_raw.csv 2>/dev/null
ncu -i $R/prof_t0_tma.ncu-rep --page source --csv --print-source sass > $O/ncu_t0_tma_sass.csv 2>/dev/null
head -24 $O/ncu_t0_tma.txt
