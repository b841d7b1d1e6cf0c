#!/bin/bash
# build a dev variant of the library: dev/build_variant.sh NAME -DFLAG ...
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -diag-suppress 177,550 "$@" \
  /root/repo/paper_2509_22681_b200/csrc/flame.cu -o /root/repo/dev/var_$name.so
