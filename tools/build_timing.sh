#!/bin/bash
# Instrumented variant of libddh.so with per-phase clock64 prints (DDH_PHASE_TIMING).
set -e
cd "$(dirname "$0")/.."
O=paper_2305_03284_b200/lib/timing; mkdir -p $O
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DDDH_PHASE_TIMING -I include"
for s in ddh_kernels.cu ddh_fused.cu; do nvcc $F -c paper_2305_03284_b200/csrc/$s -o $O/$s.o; done
nvcc $F -x cu -c paper_2305_03284_b200/csrc/ddh_api.cpp -o $O/ddh_api.cpp.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $O/libddh_timing.so $O/*.o
echo $O/libddh_timing.so
