#!/bin/bash
# Faster tuning variant: recompile one source (FILE, default kmm_tc; SRC overrides the .cu path)
# with extra flags, link against the objects of the main build (paper_2503_02259_b200/csrc/build).
# Usage: [FILE=kmm_f64] tools/build_tc_variant.sh name "-DFOO=1"   -> tools/variants/name/libkgp.so
set -e
name=$1; shift
file=${FILE:-kmm_tc}
cd "$(dirname "$0")/../paper_2503_02259_b200/csrc"
out=../../tools/variants/$name
mkdir -p $out
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Xptxas -v "$@" -c ${SRC:-$file.cu} -o $out/$file.o > $out/ptxas.log 2>&1 || (tail -30 $out/ptxas.log; false)
objs=$(ls build/*.o | grep -v "/$file.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libkgp.so $out/$file.o $objs -lcublas
rm -f $out/$file.o
echo built $out/libkgp.so
