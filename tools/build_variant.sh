#!/bin/bash
# Build an A/B variant of libmoe_b200.so with extra -D flags on tc_gemm.cu / gemv.cu:
#   tools/build_variant.sh NAME "-DMOE_TCW_RAW=2 -DMOE_TCW_B=5"
# -> build/ab/libmoe_NAME.so (select it with MOE_B200_LIB=$PWD/build/ab/libmoe_NAME.so)
set -e
name=$1; defs=$2
cd "$(dirname "$0")/../paper_2407_14417_b200/csrc"
B=../build; V=$B/abobj/$name; mkdir -p $V ../../build/ab
ARCH="-gencode arch=compute_100a,code=sm_100a"
for f in tc_gemm gemv; do
  /usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo $ARCH -Xcompiler -fPIC -I../../include -I. $defs -c kernels/$f.cu -o $V/$f.o
done
objs=$(ls $B/kernels/*.o $B/*.o $B/host/*.o | grep -v -e kernels/tc_gemm.o -e kernels/gemv.o)
/usr/local/cuda/bin/nvcc $ARCH -shared -o ../../build/ab/libmoe_$name.so $objs $V/tc_gemm.o $V/gemv.o -lcudart -ldl
echo built build/ab/libmoe_$name.so
