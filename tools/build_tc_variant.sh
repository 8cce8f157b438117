#!/bin/bash
# Faster tuning variant: recompile only kmm_tc.cu with extra flags, link against the objects
# of the main build (paper_2503_02259_b200/csrc/build). Usage: tools/build_tc_variant.sh name "-DFOO=1"
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2503_02259_b200/csrc"
out=../../tools/variants/$name
mkdir -p $out
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Xptxas -v "$@" -c ${SRC:-kmm_tc.cu} -o $out/kmm_tc.o > $out/ptxas.log 2>&1 || (tail -30 $out/ptxas.log; false)
objs=$(ls build/*.o | grep -v kmm_tc.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libkgp.so $out/kmm_tc.o $objs -lcublas
rm -f $out/kmm_tc.o
echo built $out/libkgp.so
