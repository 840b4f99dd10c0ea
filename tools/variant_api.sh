set -e
cd /root/repo
name=$1; shift
O=paper_2305_03284_b200/lib/obj; V=tools/variants; mkdir -p $V
nvcc -x cu -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -I include "$@" -c paper_2305_03284_b200/csrc/ddh_api.cpp -o $V/api_$name.o
objs=$(ls $O/*.o | grep -v ddh_api.cpp.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -Xlinker -rpath,/usr/local/cuda/lib64 -o $V/libddh_$name.so $objs $V/api_$name.o
rm $V/api_$name.o; echo $V/libddh_$name.so
