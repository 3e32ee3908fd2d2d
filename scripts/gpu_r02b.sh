# round 2, call B: sharded path + plan shards + bench contract; C3 bench (new default); dev-one-gpu 2/4/8 ranks;
# reference arm on the box; ncu DRAM bytes of the 8192^2 kernel at line blocks of 1024
mkdir -p gpurun_out/r02b
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02b
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt
timeout 900 python -m pytest tests/test_sharded_gpu.py tests/test_plan_gpu.py tests/test_bench_contract.py tests/test_p2p_gpu.py -q -x > $O/pytest_new.log 2>&1; echo pytest=$?
tail -3 $O/pytest_new.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo bench=$?
for g in 2 4 8; do
  timeout 900 python bench.py --gpus $g --dev-one-gpu --steps 3 --warmup 3 > $O/bench_c3_dev$g.json 2> $O/bench_c3_dev$g.err; echo dev$g=$?
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref_c3.json 2> $O/bench_ref_c3.err; echo ref=$?
timeout 600 python bench.py --impl reference --workload c2 --steps 2 --warmup 3 > $O/bench_ref_c2.json 2> $O/bench_ref_c2.err; echo refc2=$?
for pb in 512 1024; do
  TT_PBLOCK=$pb TT_N=8192 TT_A=180 TT_FULL=1 TT_REPS=1 TT_SAMPLER_PROF=1 timeout 600 ncu --set full --clock-control none \
    -k regex:trace_kernel -s 0 -c 1 -o $O/prof_n8192_t05_pb$pb -f python scripts/prof_c2.py > $O/prof_n8192_pb$pb.log 2>&1
  python scripts/ncu_summary.py $O/prof_n8192_t05_pb$pb.ncu-rep > $O/ncu_n8192_t05_pb$pb.txt 2>&1
  ncu -i $O/prof_n8192_t05_pb$pb.ncu-rep --page raw --csv > $O/ncu_n8192_t05_pb${pb}_raw.csv 2>/dev/null
  rm -f $O/prof_n8192_t05_pb$pb.ncu-rep
done
ls -la $O
