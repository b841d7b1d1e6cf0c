#!/bin/bash
# ncu --set full of single gemm_bf16_tcgen05 variants (dev/gemm_ab.py), reports under gpurun_out/gab/
mkdir -p gpurun_out/gab
for v in "$@"; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -c 1 -f -o gpurun_out/gab/$v \
    python dev/gemm_ab.py gpurun_out/gab/$v.json $v > gpurun_out/gab/$v.log 2>&1
done
