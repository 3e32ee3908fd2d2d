# time library variants on C2 (and C3-size n=4096 A=360)
mkdir -p gpurun_out
python scripts/time_c2.py > gpurun_out/variants.jsonl
for v in variants/*.so; do TT_LIB_PATH=$v python scripts/time_c2.py >> gpurun_out/variants.jsonl; done
TT_N=4096 TT_A=360 python scripts/time_c2.py >> gpurun_out/variants.jsonl
for v in variants/*.so; do TT_N=4096 TT_A=360 TT_LIB_PATH=$v python scripts/time_c2.py >> gpurun_out/variants.jsonl; done
cat gpurun_out/variants.jsonl
