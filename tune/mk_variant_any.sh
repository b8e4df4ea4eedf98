#!/bin/bash
# usage: tune/mk_variant_any.sh <source.cu> <out.so> <extra nvcc flags...>
# rebuilds one translation unit of paper_1902_03317_b200/csrc with extra -D flags and
# links it with the other objects into a variant library (SPT_LIB_PATH=<out.so>).
src=$1; out=$2; shift 2
base=$(basename "$src" .cu)
cd /root/repo/paper_1902_03317_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr "$@" -c $base.cu -o /tmp/${base}_var.o && \
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /root/repo/$out $(ls ../../build/csrc/*.o | grep -v /$base.o) /tmp/${base}_var.o -lcudart
