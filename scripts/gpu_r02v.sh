# round 2, call V: source-level ncu of one C3 T0-T5 launch (4096^2 / 1440)
mkdir -p gpurun_out/r02v
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02v; R=/tmp/r02v; mkdir -p $R
TT_N=4096 TT_A=1440 TT_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 -o $R/prof_c3 -f python scripts/time_c2.py > $O/prof_c3.log 2>&1; echo ncu=$?
ncu -i $R/prof_c3.ncu-rep --page source --csv --print-source sass > $O/ncu_c3_sass.csv 2>/dev/null
ncu -i $R/prof_c3.ncu-rep --page source --csv --print-source cuda > $O/ncu_c3_cuda.csv 2>/dev/null
ncu -i $R/prof_c3.ncu-rep --page raw --csv > $O/ncu_c3_raw.csv 2>/dev/null
python scripts/ncu_summary.py $R/prof_c3.ncu-rep > $O/ncu_c3.txt 2>&1
ls -la $O
