# round 2, call T: C5 sweep with the product samplers, C1/C2/C4 bench lines
mkdir -p gpurun_out/r02t
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02t
timeout 1500 python scripts/sweep.py > $O/sweep_c5.jsonl 2> $O/sweep_c5.err; echo sweep=$?
wc -l $O/sweep_c5.jsonl
timeout 600 python bench.py --workload c2 --steps 30 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err; echo c2=$?
timeout 600 python bench.py --workload c1 --steps 50 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err; echo c1=$?
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo c4=$?
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02t/bench_*.json')):
    try:
        d=json.load(open(f)); r=d['roofline']
        print(f, d['ms_per_step'], d['e2e'].get('ms_per_step'), r.get('kernel_ms'), round(r['frac'],3), d['clocks'], d.get('gpu_launches'))
    except Exception as e: print(f, 'ERR', e)
for l in open('gpurun_out/r02t/sweep_c5.jsonl'):
    d=json.loads(l); print(d['n'], d['angles'], d['functionals'], d['sampler'], round(d['ms'],3), round(d['tex_gather_frac'],3), round(d['fp32_frac'],3))
PY
