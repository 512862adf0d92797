#!/bin/bash
# Variant build of the library for A/B timing: recompiles SRC (one .cu of csrc/)
# with extra flags and links it with the regular objects of the other sources.
#   tools/build_variant.sh NAME SRC "FLAGS"   ->  build/ab/NAME/libqfuse_b200.so
set -e
NAME=$1; SRC=$2; FLAGS=$3
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OBJ=$ROOT/build/obj; OUT=$ROOT/build/ab/$NAME
mkdir -p $OUT
make -s -C $ROOT/paper_2603_02804_b200/csrc
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -diag-suppress 177 --expt-relaxed-constexpr"
$NV $FLAGS -Xptxas -v -c -o $OUT/${SRC%.cu}.o $ROOT/paper_2603_02804_b200/csrc/$SRC 2> $OUT/ptxas.txt
OBJS=$(ls $OBJ/*.o | grep -v "/${SRC%.cu}.o$")
$NV -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -Xlinker -rpath,/usr/local/cuda/lib64 \
  -o $OUT/libqfuse_b200.so $OBJS $OUT/${SRC%.cu}.o -ldl
grep -E "registers|spill" $OUT/ptxas.txt | head -4
