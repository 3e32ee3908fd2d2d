# round 2, call AK: randomised parity stress of this build (all three samplers, TMA Radon included)
mkdir -p gpurun_out/r02ak
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02ak
for seed in 1 2 3 4; do timeout 1200 python scripts/parity_stress.py 1500 $seed; done > $O/parity_stress.txt 2>&1
cat $O/parity_stress.txt
