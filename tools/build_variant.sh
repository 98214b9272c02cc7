#!/bin/bash
# Build an A/B variant of libinfllm2.so with extra -D flags on one source:
#   tools/build_variant.sh <out.so> <source.cu> -DFOO=1 ...
# then time it with INFLLM2_LIB_PATH=<out.so> python ...
set -e
out=$1; src=$2; shift 2
base=$(basename $src .cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Iinclude -Ipaper_2506_07900_b200/csrc "$@" -c $src -o build/alt/$base.o
objs=$(ls build/*.o | grep -v "/$base.o" | grep -v attend_tc2)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $objs build/alt/$base.o
