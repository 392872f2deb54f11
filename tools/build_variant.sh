#!/bin/bash
# build a tuning variant of libsdnn.so: tools/build_variant.sh NAME -DFLAG=V ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p variants
gcc -O3 -std=gnu11 -fPIC -c -o /tmp/sdnn_gen_$name.o paper_1909_05631_b200/csrc/sdnn_gen.c
gcc -O3 -std=gnu11 -fPIC -mavx2 -fopenmp -c -o /tmp/sdnn_host_$name.o paper_1909_05631_b200/csrc/sdnn_host.c
/usr/local/cuda/bin/nvcc -gencode=arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared \
  -Xcompiler -fPIC,-fopenmp,-mavx2 -cudart static "$@" -o variants/libsdnn_$name.so \
  paper_1909_05631_b200/csrc/sdnn.cu /tmp/sdnn_gen_$name.o /tmp/sdnn_host_$name.o -lpthread -lgomp
