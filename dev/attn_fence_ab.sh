# interleaved bench A/B of attention compiler-barrier variants (dev/build_variant.sh aprobeM -DFLAME_ATTN_PROBE_MASK=M)
for r in 1 2; do
  for lib in paper_2509_22681_b200/_flame_b200.so dev/var_aprobe3.so dev/var_aprobe12.so dev/var_aprobe15.so; do
    FLAME_B200_LIB=$lib timeout 300 python bench.py --workload ${1:-cfg3} --no-cpu-baseline --no-fp32-line 2>/dev/null | tail -1 > gpurun_out/af_$(basename $lib .so)_${1:-cfg3}_$r.json
  done
done
