#!/bin/bash
# build_var.sh <tag> <extra nvcc flags...>: a variant of the library under tools/libvar/lib_<tag>.so
# (only leaf_fast.cu is rebuilt with the extra flags; the other objects come from build/)
set -e
tag=$1; shift
mkdir -p tools/libvar build/var_$tag
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC "$@" \
  -c paper_1302_6945_b200/csrc/leaf_fast.cu -o build/var_$tag/leaf_fast.o
objs=$(ls build/*.o | grep -v leaf_fast.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/libvar/lib_$tag.so $objs build/var_$tag/leaf_fast.o -lcudart
echo built tools/libvar/lib_$tag.so
