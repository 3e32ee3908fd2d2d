for cfg in "1024 720" "2048 180" "4096 90"; do
  set -- $cfg
  for ns in 16 32 64 128; do
    TT_SLOTS_PER_LINE=$ns TT_N=$1 TT_A=$2 python scripts/time_c2.py | sed "s/^/ns=$ns /"
  done
done
