#!/bin/bash
# Tuning builds of libfzb200.so with lorenzo.cu compiled under extra -D flags:
#   scripts/build_var.sh NAME "-DFOO=1 ..."  -> paper_2509_20563_b200/_build/var/libfzb200_NAME.so
set -e
cd "$(dirname "$0")/../paper_2509_20563_b200"
mkdir -p _build/var
for f in lorenzo huffman; do
    nvcc $2 -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
        --expt-relaxed-constexpr -I ../include -c csrc/$f.cu -o _build/var/${f}_$1.o
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o _build/var/libfzb200_$1.so _build/stream_ops.o \
    _build/var/lorenzo_$1.o _build/interp.o _build/bitshuffle.o _build/var/huffman_$1.o _build/dualquant.o -lcudart
rm -f _build/var/lorenzo_$1.o _build/var/huffman_$1.o
