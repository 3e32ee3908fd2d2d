# round 2, call CY: HEAD sanity -- default bench line and the 2-rank one-GPU p2p path through bench.py
O=gpurun_out/r02cy
mkdir -p $O
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo bench=$?
timeout 600 python bench.py --gpus 2 --workload c3 --dev-one-gpu --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3_dev2.json 2> $O/bench_c3_dev2.err; echo dev2=$?
python -c "
import json
d=json.load(open('$O/bench_c3.json')); print('c3', d['ms_per_step'], d['value'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['clocks'])
d=json.load(open('$O/bench_c3_dev2.json')); print('dev2', d.get('e2e_matches_device_result'), d['config']['parallelism'])"
