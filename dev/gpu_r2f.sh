#!/bin/bash
O=gpurun_out/r2f; mkdir -p $O
for w in cfg4 cfg3; do
timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$w.log 2>&1; tail -1 $O/bench_$w.log > $O/bench_$w.json
python -c "
import json; d=json.load(open('$O/bench_$w.json')); r=d['roofline']
print('$w', d['value'], d['e2e']['value'], r['kernel'], r['frac'], r['avg_launch_ms'])
for k,v in d['kernels'].items(): print('  ', k, v)"
done
