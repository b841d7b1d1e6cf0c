#!/bin/bash
# W1 (GELU epilogue) variants: libraries x single CTA / CTA pairs
mkdir -p gpurun_out/gm; VARIANT=${VARIANT:-w1_bias_gelu}
for lib in paper_2509_22681_b200/_flame_b200.so "$@"; do
  for mink in 1024 512; do
    tag=$(basename $lib .so)_mink${mink}_$VARIANT
    FLAME_B200_LIB=$lib FLAME_GEMM_PAIR_MINK=$mink python dev/gemm_ab.py gpurun_out/gm/$tag.json $VARIANT > /dev/null 2>&1
    echo "$tag $(cat gpurun_out/gm/$tag.json)"
  done
done
