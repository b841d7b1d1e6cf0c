#!/bin/bash
# interleaved A/B over environment settings: each arg is "default" or VAR=VALUE; 3 rounds
mkdir -p gpurun_out
for rep in 1 2 3; do
  for e in "$@"; do
    if [ "$e" = "default" ]; then envs=""; else envs="$e"; fi
    env $envs timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/abenv.log 2>&1
    tail -1 gpurun_out/abenv.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('$e'.ljust(26), 'ms %.4f'%d['ms_per_step'], ' '.join('%s=%.4f'%(n[5:12],v['ms_per_step']) for n,v in sorted(k.items()) if n.startswith('gemm')))"
  done
done
