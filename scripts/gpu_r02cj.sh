# round 2, call CJ: C5 sweep of the final build
O=gpurun_out/r02cj
mkdir -p $O
timeout 1500 python scripts/sweep.py > $O/sweep_c5.jsonl 2> $O/sweep_c5.err; echo sweep=$?
wc -l $O/sweep_c5.jsonl
