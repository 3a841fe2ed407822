#!/bin/bash
# Build an experimental variant of the library with extra nvcc flags on smnn_rf.cu / smnn_pipe.cu:
#   tools/build_variant.sh <tag> "<flags>"   ->  paper_2410_06074_b200/lib/libsmnn_v_<tag>.so (load with SMNN_LIB=...)
set -e
cd "$(dirname "$0")/../paper_2410_06074_b200/csrc"
tag=$1; shift; fl="$*"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I ../../include -I ."
nvcc $F -c -o /tmp/rf_$tag.o smnn_rf.cu $fl &
nvcc $F -c -o /tmp/pipe_$tag.o smnn_pipe.cu $fl &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o ../lib/libsmnn_v_$tag.so ../lib/smnn_kernels.o /tmp/rf_$tag.o /tmp/pipe_$tag.o
echo ../lib/libsmnn_v_$tag.so
