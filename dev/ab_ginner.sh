mkdir -p gpurun_out
for m in 0 1; do
  FLAME_GEMM_GINNER=$m timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum --cache-control none --clock-control none --kernel-name-base mangled -k regex:5flame -c 11 --csv python dev/prof_step.py cfg3 1 1 > gpurun_out/ab_ginner_$m.csv 2>/dev/null
done
