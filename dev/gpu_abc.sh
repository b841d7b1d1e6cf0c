#!/bin/bash
# interleaved multi-variant bench: each arg is a lib path ("" = default build); 3 rounds
mkdir -p gpurun_out
for rep in 1 2 3; do
  for lib in "$@"; do
    if [ "$lib" = "default" ]; then unset FLAME_B200_LIB; else export FLAME_B200_LIB=$lib; fi
    timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/abc.log 2>&1
    tail -1 gpurun_out/abc.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('$lib'.ljust(20), 'ms %.4f'%d['ms_per_step'], ' '.join('%s=%.4f'%(n[:10],v['ms_per_step']) for n,v in sorted(k.items())))"
  done
done
