# round 2, call ZA: ncu of one C2 T0-T5 launch (1024^2 / 720) for profiles/ncu_c2_summary.json + GPU suite
mkdir -p gpurun_out/r02za
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02za; R=/tmp/r02za; mkdir -p $R
TT_N=1024 TT_A=720 TT_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 -o $R/prof_c2 -f python scripts/time_c2.py > $O/prof_c2.log 2>&1; echo ncu=$?
ncu -i $R/prof_c2.ncu-rep --page raw --csv > $O/ncu_c2_raw.csv 2>/dev/null
python scripts/ncu_summary.py $R/prof_c2.ncu-rep > $O/ncu_c2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest_gpu=$?
tail -3 $O/pytest_gpu.log
ls -la $O
