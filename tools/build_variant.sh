#!/bin/bash
# Build an experimental variant of the library with extra nvcc flags (compile-time macros only):
#   tools/build_variant.sh <tag> "<flags>"   ->  paper_2410_06074_b200/lib/variants/libsmnn_<tag>.so
# Measurement tools load it explicitly (tools/path_sweep.py --lib ...); the product never does.
set -e
cd "$(dirname "$0")/../paper_2410_06074_b200/csrc"
tag=$1; shift; fl="$*"
mkdir -p ../lib/variants
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I ../../include -I ."
for s in smnn_kernels smnn_rf smnn_pipe smnn_x64; do
  nvcc $F -c -o /tmp/${s}_$tag.o $s.cu $fl &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o ../lib/variants/libsmnn_$tag.so \
  /tmp/smnn_kernels_$tag.o /tmp/smnn_rf_$tag.o /tmp/smnn_pipe_$tag.o /tmp/smnn_x64_$tag.o
echo ../lib/variants/libsmnn_$tag.so
