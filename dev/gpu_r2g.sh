#!/bin/bash
O=gpurun_out/r2g; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/all.log 2>&1; echo rc=$? >> $O/all.log; tail -3 $O/all.log
for w in cfg4 cfg1 cfg3; do
timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-fp32-line > $O/bench_$w.log 2>&1; tail -1 $O/bench_$w.log > $O/bench_$w.json
python -c "
import json; d=json.load(open('$O/bench_$w.json')); print('$w', d['value'], 'e2e', d['e2e']['value'], d['e2e'].get('request_p99_ms'), d.get('p99_ms'))"
done
