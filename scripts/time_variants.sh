# time every variants/lib_*.so on C2 (TT_N/TT_A override) with scripts/time_c2.py
for f in variants/lib_*.so; do
  TT_LIB_PATH=$f timeout 300 python scripts/time_c2.py
done
