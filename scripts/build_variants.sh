# build experimental library variants (one schedule, -D knobs) into variants/ in parallel
# usage: bash scripts/build_variants.sh NAME "-DKNOB=V ..." [NAME "-D..."]...
mkdir -p variants
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  ( nvcc -ccbin g++ -shared -Xcompiler -fPIC,-ffp-contract=off -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo \
      -std=c++17 -Iinclude -DTT_DEV_ONLY_SLOTS=${SLOTS:-32} $defs paper_1604_03410_b200/csrc/tt_kernels.cu \
      paper_1604_03410_b200/csrc/tt_context.cpp paper_1604_03410_b200/csrc/tt_device_api.cpp paper_1604_03410_b200/csrc/tt_host.cpp paper_1604_03410_b200/csrc/tt_jit.cpp -ldl -o variants/lib_$name.so \
      && echo built $name ) &
done
wait
