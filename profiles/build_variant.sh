#!/bin/bash
# Build an experiment variant of the library: build/<name>.so with extra nvcc
# defines (A/B runs copy it over paper_2110_14934_b200/librgbdseg_b200.so on
# the GPU box).   usage: profiles/build_variant.sh NAME "-DX=1 -DY=2"
set -e
cd "$(dirname "$0")/.."
N=$1; shift
mkdir -p build/$N
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true -ftz=false -Xcompiler -fPIC,-O2 $*"
nvcc $F -c paper_2110_14934_b200/csrc/rgbdseg_kernels.cu -o build/$N/k.o -Xptxas -v 2> build/$N/ptxas.log &
nvcc $F -c paper_2110_14934_b200/csrc/rgbdseg_capi.cu -o build/$N/c.o
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -o build/$N.so build/$N/k.o build/$N/c.o
grep -A1 "k_fused_ldgILi5ELi5ELb1ELb0ELb0E" build/$N/ptxas.log | grep -o "[0-9]* bytes spill stores\|Used [0-9]* registers" | head -2 | tr '\n' ' '; echo " <- $N"
