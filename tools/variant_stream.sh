#!/bin/bash
# Build a libddh.so variant that differs only in ddh_stream.cu compile flags:
#   tools/variant_stream.sh NAME -DFOO=1 ...   -> tools/variants/libddh_NAME.so
# (needs the regular build's objects in paper_2305_03284_b200/lib/obj)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
O=paper_2305_03284_b200/lib/obj; V=tools/variants; mkdir -p $V
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -I include "$@" \
  -c paper_2305_03284_b200/csrc/ddh_stream.cu -o $V/stream_$name.o
objs=$(ls $O/*.o | grep -v ddh_stream.cu.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -Xlinker -rpath,/usr/local/cuda/lib64 -o $V/libddh_$name.so $objs $V/stream_$name.o
rm $V/stream_$name.o
echo $V/libddh_$name.so
