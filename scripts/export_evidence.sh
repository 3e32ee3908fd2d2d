# copy a gpu_full.sh (+ gpu_big.sh) run from gpurun_out/ into profiles/ (round-tagged names)
set -e
R=${ROUND:-r01}
G=gpurun_out
P=profiles
cp $G/bench.json $P/${R}_bench_c2.json
cp $G/bench_ref.json $P/${R}_bench_reference_c2.json
cp $G/launches_c2.csv $P/${R}_launches_c2.csv
cp $G/sweep.jsonl $P/${R}_sweep_c5.jsonl
ncu -i $G/prof_c2.ncu-rep --page details --csv > $P/${R}_ncu_c2_trace_details.csv 2>/dev/null
ncu -i $G/prof_c2.ncu-rep --page raw --csv > $P/${R}_ncu_c2_trace_raw.csv 2>/dev/null
ncu -i $G/prof_c2.ncu-rep --page source --csv --print-source cuda,sass > $G/cs_c2.csv 2>/dev/null
python scripts/ncu_lines.py $G/cs_c2.csv 40 > $P/${R}_ncu_c2_trace_lines.txt
ncu -i $G/prof_circus.ncu-rep --page details --csv > $P/${R}_ncu_c2_circus_details.csv 2>/dev/null
for t in n8192_t0 n8192_t05; do
  if [ -f $G/ncu_$t.txt ]; then cp $G/ncu_$t.txt $P/${R}_ncu_${t}_summary.txt; fi
done
if [ -f $G/ncu_n8192_t0_raw.csv ]; then cp $G/ncu_n8192_t0_raw.csv $P/${R}_ncu_n8192_t0_raw.csv; fi
python scripts/ncu_summary.py $G/prof_c2.ncu-rep
