# round 2, call AX: final evidence (128-tap TMA stages) -- GPU suite, smoke, C5 sweep, C3 bench + launch list
mkdir -p gpurun_out/r02ax
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02ax
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo pytest_gpu=$?
tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 1500 python scripts/sweep.py > $O/sweep_c5.jsonl 2> $O/sweep_c5.err; echo sweep=$?
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
cut -c1-300 $O/bench_c3.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launches_c3.log 2>&1; echo ncu_launches=$?
python - <<'PY'
import json
for l in open('gpurun_out/r02ax/sweep_c5.jsonl'):
    d=json.loads(l)
    if d['functionals']=='T0': print(d['n'], d['angles'], d['sampler'], round(d['ms'],3), round(d['tex_gather_frac'],3))
PY
