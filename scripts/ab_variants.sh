for cfg in "1024 720 1" "256 360 1" "512 360 1" "2048 720 1" "4096 1440 0"; do
  set -- $cfg
  for f in variants/lib_*.so; do
    echo -n "$f n=$1 A=$2 full=$3 "; TT_N=$1 TT_A=$2 TT_FULL=$3 TT_LIB_PATH=$f timeout 300 python scripts/time_c2.py
  done
done
