#!/bin/bash
# loadgen ablations at the cfg3 model (d=512, 8 blocks) on one B200: CSV reports
# in gpurun_out/loadgen/; scenario x (cache, mem_opt, routing)
mkdir -p gpurun_out/loadgen
run() {  # scenario cache mem_opt routing concurrency duration
  timeout 900 python -m paper_2509_22681_b200.loadgen --config dev/configs/service_cfg3.json --scenario $1 \
    --cache $2 --mem-opt $3 --routing $4 --concurrency $5 --duration $6 \
    --out gpurun_out/loadgen/$1_cache-$2_mem-$3_$4_c$5.csv 2>&1 | tail -1
}
run mixed on on explicit 32 20
run mixed on on explicit 8 20
run long on on explicit 32 15
run base on on explicit 32 15
run mixed off on explicit 32 15
run mixed on off explicit 32 15
run mixed on on implicit 8 15
