#!/bin/bash
# Builds an experiment variant of the library with the fused kernel compiled
# under extra flags:  scripts/build_exp.sh <name> [nvcc -D flags...]
#   -> paper_2204_01722_b200/exp/lib_<name>.so   (load with HXG_LIBRARY=...)
set -e
cd "$(dirname "$0")/../paper_2204_01722_b200/csrc"
make -j8 >/dev/null
NAME=$1; shift
UNIT=${UNIT:-fused_apply}    # translation unit rebuilt with the flags
SRC=${SRC:-$UNIT.cu}         # alternative source for it (e.g. an older version)
B=../../build/exp_$NAME; mkdir -p $B ../exp
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
  -I../../include -I. --expt-relaxed-constexpr "$@" -x cu -c $SRC -o $B/$UNIT.o
OBJS=$(ls ../../build/csrc/*.o | grep -v "/$UNIT.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../exp/lib_$NAME.so $B/$UNIT.o $OBJS \
  -lcusolver -lcusparse -lcublas -lcudart
echo built exp/lib_$NAME.so
