mkdir -p gpurun_out
for i in 1 2; do
python scripts/time_c2.py
for v in variants/*.so; do TT_LIB_PATH=$v python scripts/time_c2.py; done
done
