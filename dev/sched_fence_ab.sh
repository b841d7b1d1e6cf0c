set -u
run() { # tag lib bn workload
  FLAME_B200_LIB=$2 FLAME_GATED_BN=$3 timeout 300 python bench.py --workload $4 --no-cpu-baseline --no-fp32-line 2>/dev/null | tail -1 > gpurun_out/sf_$1_$4.json
}
for r in 1 2; do
  run base128_r$r dev/var_probe0.so 128 cfg3
  run fence128_r$r paper_2509_22681_b200/_flame_b200.so 128 cfg3
  run fence256_r$r paper_2509_22681_b200/_flame_b200.so 256 cfg3
done
for w in cfg5 cfg2; do
  run base128 dev/var_probe0.so 128 $w
  run fence128 paper_2509_22681_b200/_flame_b200.so 128 $w
  run fence256 paper_2509_22681_b200/_flame_b200.so 256 $w
done
