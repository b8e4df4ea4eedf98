#!/bin/bash
out=$1; shift
cd /root/repo/paper_1902_03317_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr "$@" -c ttv.cu -o /tmp/tv_var.o && \
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /root/repo/$out $(ls ../../build/csrc/*.o | grep -v /ttv.o) /tmp/tv_var.o -lcudart
