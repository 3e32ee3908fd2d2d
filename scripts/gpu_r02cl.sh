# round 2, call CL: kernel-only durations of the TMA Radon launch at 1024^2/180 (one vs two line blocks per CTA)
O=gpurun_out/r02cl
mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
TT_SAMPLER_ID=2 TT_N=1024 TT_A=180 TT_FULL=0 TT_REPS=3 timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none --csv python scripts/time_c2.py > $O/ncu_1024_180.csv 2>&1
TT_SAMPLER_ID=1 TT_N=1024 TT_A=180 TT_FULL=0 TT_REPS=30 timeout 120 python scripts/time_c2.py > $O/tex_1024_180.json 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r02cl/ncu_1024_180.csv')) if len(r)>10 and r[0]!='ID']
for r in rows: print(r[4][:40], r[12], r[14])
PY
tail -1 $O/tex_1024_180.json
