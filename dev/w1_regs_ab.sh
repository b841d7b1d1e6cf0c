# interleaved bench A/B: W1 epilogue with setmaxnreg + fully unrolled chunk loop (dev/var_w1big.so) vs the default
for r in 1 2; do
  for lib in paper_2509_22681_b200/_flame_b200.so dev/var_w1big.so; do
    for w in cfg3 cfg5 cfg2; do
      FLAME_B200_LIB=$lib timeout 300 python bench.py --workload $w --no-cpu-baseline --no-fp32-line 2>/dev/null | tail -1 > gpurun_out/w1r_$(basename $lib .so)_${w}_$r.json
    done
  done
done
