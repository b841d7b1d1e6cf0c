# interleaved bench A/B: async (cp.async, double-buffered) vs synchronous GEMM column-vector staging
for r in 1 2; do
  for lib in paper_2509_22681_b200/_flame_b200.so dev/var_cvsync.so; do
    for w in cfg3 cfg5; do
      FLAME_B200_LIB=$lib timeout 300 python bench.py --workload $w --no-cpu-baseline --no-fp32-line 2>/dev/null | tail -1 > gpurun_out/cv_$(basename $lib .so)_${w}_$r.json
    done
  done
done
