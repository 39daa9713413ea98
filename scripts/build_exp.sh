#!/bin/bash
# Builds an experiment variant of the library (fused kernel compiled with
# -DHXG_EXPERIMENT=$1) as paper_2204_01722_b200/libhexmg_b200_exp$1.so.
set -e
cd "$(dirname "$0")/../paper_2204_01722_b200/csrc"
make -j8 >/dev/null
E=$1
B=../../build/exp$E; mkdir -p $B
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
  -I../../include -I. --expt-relaxed-constexpr -DHXG_EXPERIMENT=$E $EXTRA -c fused_apply.cu -o $B/fused_apply.o
OBJS=$(ls ../../build/csrc/*.o | grep -v fused_apply.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libhexmg_b200_exp$E.so $B/fused_apply.o $OBJS \
  -lcusolver -lcusparse -lcublas -lcudart
echo built ../libhexmg_b200_exp$E.so
