#!/bin/bash
# Full-library experiment build with extra -D flags (layout macros reach every
# kernel):  scripts/build_full_exp.sh <name> [-D...]  -> paper_2204_01722_b200/exp/lib_<name>.so
set -e
cd "$(dirname "$0")/../paper_2204_01722_b200/csrc"
NAME=$1; shift
B=../../build/full_$NAME; mkdir -p $B ../exp
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I../../include -I. --expt-relaxed-constexpr"
for f in operator fused_apply transfer vector coarse ndchol; do nvcc $F "$@" -c $f.cu -o $B/$f.o 2>/dev/null & done
for f in setup solver capi; do nvcc $F "$@" -x cu -c $f.cpp -o $B/$f.o 2>/dev/null & done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../exp/lib_$NAME.so $B/*.o -lcusolver -lcusparse -lcublas -lcudart
echo built exp/lib_$NAME.so
