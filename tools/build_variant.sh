#!/bin/bash
# Build a variant library for same-box A/B: recompile ONE source with extra flags and
# relink it with the other objects of the current build.
# usage: tools/build_variant.sh <source.cu> <out-suffix> [extra nvcc flags...]
cd "$(dirname "$0")/.."
src=$1; suf=$2; shift 2
L=paper_2302_03213_b200/_lib
obj=/tmp/variant_$suf.o
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr -I include "$@" -c paper_2302_03213_b200/csrc/$src -o $obj || exit 1
objs=$(ls $L/*.o | grep -v "/${src%.cu}.o")
nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs $obj -o $L/liblutgpu_$suf.so \
  -Xlinker --version-script=$L/exports.map -lcudart_static -lrt -ldl -lpthread && echo "built $L/liblutgpu_$suf.so"
