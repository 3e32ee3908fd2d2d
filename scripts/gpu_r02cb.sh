# round 2, call CB: which half of the tap-range clip costs time on T0-T5 (pass 1 vs pass 2), C3 and C2 schedules
mkdir -p gpurun_out/r02cb
O=gpurun_out/r02cb
export PATH=/usr/local/cuda/bin:$PATH
for v in c3_noclip c3_clip c3_p1only c3_p2only; do TT_LIB_PATH=variants/lib_$v.so TT_N=4096 TT_A=1440 TT_REPS=3 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"; done > $O/ab.txt 2>&1
for v in c2_noclip c2_clip c2_p1only c2_p2only; do TT_LIB_PATH=variants/lib_$v.so TT_N=1024 TT_A=720 TT_REPS=20 timeout 300 python scripts/time_c2.py 2>&1 | tail -1 | sed "s/^/$v /"; done >> $O/ab.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02cb/ab.txt'):
    v,j=l.split(' ',1)
    try: d=json.loads(j); print(v,d['n'],d['A'],round(d['median_ms'],4), d['checksum'])
    except Exception: print(l[:150])
PY
for v in c2_noclip c2_clip; do
TT_LIB_PATH=variants/lib_$v.so TT_N=1024 TT_A=720 TT_REPS=1 timeout 600 ncu --clock-control none -k regex:trace_kernel -c 1 --csv --metrics smsp__inst_executed.sum,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__thread_inst_executed.sum python scripts/time_c2.py > $O/ncu_$v.csv 2>&1
grep -v "^==" $O/ncu_$v.csv | tail -8
done
