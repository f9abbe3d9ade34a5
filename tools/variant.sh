#!/bin/bash
# Build a variant of libnegf_b200.so with extra nvcc flags for A/B timing:
#   tools/variant.sh <name> <flags...>   -> build/variants/<name>.so (load with NEGF_LIB=...)
set -e
cd /root/repo
name=$1; shift
out=build/variants/$name
mkdir -p $out
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC,-O3 -Iinclude"
objs=""
for s in tree.cpp plan.cpp kernels.cu capi.cu lead.cu output.cpp; do
  $NV "$@" -c paper_1305_1070_b200/csrc/$s -o $out/$s.o
  objs="$objs $out/$s.o"
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/variants/$name.so $objs -ldl -lpthread -lrt
echo build/variants/$name.so
