#!/bin/bash
# Build a tuning variant of libkgp.so with extra nvcc flags into tools/variants/<name>/
# (run it with KGP_LIB=tools/variants/<name>/libkgp.so). Usage: tools/build_variant.sh name "-DFOO=1 ..."
set -e
name=$1; shift
flags="$*"
cd "$(dirname "$0")/../paper_2503_02259_b200/csrc"
out=../../tools/variants/$name
mkdir -p $out
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $flags"
for f in kgp_api kmm_tc kmm_f64 prep panels woodbury pcg afn symv wgemm; do
  $NV -c $f.cu -o $out/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libkgp.so $out/*.o -lcublas
rm -f $out/*.o
echo built $out/libkgp.so
