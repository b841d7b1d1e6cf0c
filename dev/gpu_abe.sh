#!/bin/bash
# interleaved env-variant bench: each arg is an env assignment list ("-" = none); 3 rounds
mkdir -p gpurun_out
for rep in 1 2 3; do
  for e in "$@"; do
    if [ "$e" = "-" ]; then envs=""; else envs="$e"; fi
    env $envs timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/abe.log 2>&1
    tail -1 gpurun_out/abe.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('$e'.ljust(40), 'ms %.4f'%d['ms_per_step'], ' '.join('%s=%.4f'%(n[:10],v['ms_per_step']) for n,v in sorted(k.items())))"
  done
done
