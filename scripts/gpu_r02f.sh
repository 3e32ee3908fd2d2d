# round 2, call F: fused P stage variants on C2 (time + ncu of the default), C3 slot variants
mkdir -p gpurun_out/r02f
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02f
for v in v0 v1 v2 v3; do
  for c in 0 1; do
    TT_LIB_PATH=vlibs/lib_$v.so TT_CIRC=$c TT_REPS=10 timeout 300 python scripts/time_c2.py | sed "s/^/$v circ=$c /"
  done
done > $O/epi_variants.txt 2>&1
cat $O/epi_variants.txt
TT_CIRC=1 TT_A=72 TT_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 \
  -o $O/prof_c2_circ -f python scripts/time_c2.py > $O/prof_c2_circ.log 2>&1
python scripts/ncu_summary.py $O/prof_c2_circ.ncu-rep > $O/ncu_c2_circ.txt 2>&1
for sl in 64 128 256; do
  TT_SLOTS_PER_LINE=$sl TT_N=4096 TT_A=1440 TT_REPS=3 timeout 300 python scripts/time_c2.py | sed "s/^/slots=$sl /"
done > $O/c3_slots.txt 2>&1
cat $O/c3_slots.txt
ls -la $O
