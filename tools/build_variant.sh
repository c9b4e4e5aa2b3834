#!/bin/bash
# Build an A/B variant of libcgbn.so with extra compile-time knobs, in-tree (it travels to
# the GPU box with the repo); select it at run time with CGBN_LIB.
#   tools/build_variant.sh minb3 -DCGBN_CT_MINB=3   ->  paper_1711_07240_b200/libcgbn_minb3.so
set -eu
name=$1; shift
B=build/var_$name
mkdir -p $B
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr -Xptxas -v $*"
S=paper_1711_07240_b200/csrc
nvcc $F -c -o $B/a0.o $S/cgbn.cu 2> $B/ptxas_a0.log &
nvcc $F -c -o $B/a1.o $S/cgbn_bf16.cu 2> $B/ptxas_a1.log &
nvcc $F -c -o $B/a2.o $S/cgbn_f16.cu 2> $B/ptxas_a2.log &
nvcc $F -c -o $B/conv.o $S/cgbn_conv.cu 2> $B/ptxas_conv.log &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1711_07240_b200/libcgbn_$name.so $B/a0.o $B/a1.o $B/a2.o $B/conv.o
echo "built paper_1711_07240_b200/libcgbn_$name.so"
