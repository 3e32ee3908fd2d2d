# round 2, call AN: ncu of the C1 kernel (256^2 / 360, T0-T5)
mkdir -p gpurun_out/r02an
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02an; R=/tmp/r02an; mkdir -p $R
TT_N=256 TT_A=360 TT_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 -o $R/prof_c1 -f python scripts/time_c2.py > $O/prof_c1.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py $R/prof_c1.ncu-rep > $O/ncu_c1.txt 2>&1
ncu -i $R/prof_c1.ncu-rep --page raw --csv > $O/ncu_c1_raw.csv 2>/dev/null
head -40 $O/ncu_c1.txt
