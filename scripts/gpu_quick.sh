mkdir -p gpurun_out
python scripts/time_c2.py
TT_N=256 TT_A=360 python scripts/time_c2.py
timeout 600 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python -c "import json; j=json.load(open('gpurun_out/bench_c2.json')); print('bench c2 ms', j['ms_per_step'], 'kernel', j['roofline']['kernel_ms'], 'frac', j['roofline']['frac'], 'e2e', j['e2e']['ms_per_step'])"
