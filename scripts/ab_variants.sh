# A/B timing of every variants/lib_*.so with scripts/time_c2.py over a few configurations
# (CFGS="n A full;..." overrides the default list)
CFGS=${CFGS:-"1024 720 1;256 360 1;512 360 1;2048 720 1;4096 1440 0"}
IFS=';' read -ra LIST <<< "$CFGS"
for cfg in "${LIST[@]}"; do
  set -- $cfg
  for f in variants/lib_*.so; do
    echo -n "$(basename $f) n=$1 A=$2 full=$3 "
    TT_N=$1 TT_A=$2 TT_FULL=$3 TT_LIB_PATH=$f timeout 300 python scripts/time_c2.py | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['median_ms'],4), d['checksum'])"
  done
done
