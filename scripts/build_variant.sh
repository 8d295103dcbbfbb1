#!/bin/bash
# build_variant.sh <decode.cu> <out.so> [extra nvcc flags...]  (development experiments only)
set -e
cd "$(dirname "$0")/.."
SRC=$1; OUT=$2; shift 2
mkdir -p build/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include -I paper_2512_19179_b200/csrc \
  -Xcompiler -fPIC,-ffp-contract=off,-fno-fast-math "$@" -c $SRC -o build/variants/$(basename $OUT).o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT build/variants/$(basename $OUT).o \
  build/l4/l4_migrate.cu.o build/l4/l4_common.cpp.o build/l4/l4_pool.cpp.o build/l4/l4_partition.cpp.o -lpthread -ldl -lrt
