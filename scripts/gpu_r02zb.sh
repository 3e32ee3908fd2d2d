# round 2, call ZB: schedule width (slots per line, TT_SLOTS_PER_LINE) at C1 / C2 / C3 / 2048^2 -- timing only
mkdir -p gpurun_out/r02zb
O=gpurun_out/r02zb
for cfg in "256 360 8" "256 360 16" "256 360 32" "1024 720 32" "1024 720 64" "2048 720 64" "2048 720 128" "4096 1440 64" "4096 1440 128" "4096 1440 256"; do
  set -- $cfg
  echo "slots=$3 $(TT_N=$1 TT_A=$2 TT_REPS=5 TT_SLOTS_PER_LINE=$3 timeout 300 python scripts/time_c2.py 2>&1 | tail -1)" >> $O/slots.txt
done
cat $O/slots.txt
