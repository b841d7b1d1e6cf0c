#!/bin/bash
# one gemm_ab variant across library builds, interleaved: dev/gemm_ab_libs.sh VARIANT ROUNDS LIB...
v=$1; n=$2; shift 2
mkdir -p gpurun_out/gl
for r in $(seq $n); do
  for lib in "$@"; do
    FLAME_B200_LIB=$lib python dev/gemm_ab.py gpurun_out/gl/tmp.json $v > /dev/null 2>&1
    echo "$(basename $lib .so) $v $(cat gpurun_out/gl/tmp.json)"
  done
done
