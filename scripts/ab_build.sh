#!/usr/bin/env bash
# A/B experiments: link libtang with one source replaced -> variants/libtang_<tag>.so
# usage: scripts/ab_build.sh TAG SOURCE_NAME REPLACEMENT.cu   (run after __graft_entry__.build())
set -e
TAG=$1; SRC=$2; REP=$3
ROOT=$(cd "$(dirname "$0")/.." && pwd)
B=$ROOT/paper_2601_03187_b200/_build
mkdir -p $ROOT/variants
cp "$REP" $ROOT/paper_2601_03187_b200/csrc/_ab_$TAG.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I $ROOT/include \
     --expt-relaxed-constexpr -c $ROOT/paper_2601_03187_b200/csrc/_ab_$TAG.cu -o $ROOT/variants/_ab_$TAG.o
rm $ROOT/paper_2601_03187_b200/csrc/_ab_$TAG.cu
OBJS=$(ls $B/*.o | grep -v "/$SRC.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $ROOT/variants/libtang_$TAG.so $OBJS $ROOT/variants/_ab_$TAG.o
echo $ROOT/variants/libtang_$TAG.so
