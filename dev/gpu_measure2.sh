#!/bin/bash
# round-2 measurement: bench lines (cfg3 with fp32 line, cfg4, cfg2, cfg5, cfg1), sustained cfg3,
# reference arm, ncu launch list + full capture of the bench's own cfg3 pass
O=gpurun_out/${MEASURE_OUT:-m2}; mkdir -p $O
for w in cfg3 cfg4 cfg2 cfg5 cfg1; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > $O/bench_$w.log 2>&1
  tail -1 $O/bench_$w.log > $O/bench_$w.json
done
timeout 900 python bench.py --workload cfg3 --steps 150 --warmup 5 --no-cpu-baseline --no-fp32-line > $O/bench_cfg3_sustained.log 2>&1
tail -1 $O/bench_cfg3_sustained.log > $O/bench_cfg3_sustained.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_cfg3.log 2>&1; tail -1 $O/ref_cfg3.log > $O/ref_cfg3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 18 -c 9 --csv \
  --log-file $O/launches_cfg3.csv python tools/prof_step.py cfg3 3 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:5flame -c 9 -o $O/prof_full_cfg3 -f python tools/prof_step.py cfg3 1 > $O/ncu_full.log 2>&1
for w in cfg3 cfg4 cfg2 cfg5 cfg1; do python -c "
import json; d=json.load(open('$O/bench_$w.json')); print('$w', round(d['value']/1e6,3), 'M/s e2e', round(d['e2e']['value']/1e6,3), 'p99', round(d['p99_ms'],2), 'roof', d['roofline']['kernel'], d['roofline']['frac'], 'cpu', (d.get('cpu_baseline') or {}).get('value'), 'fp32', (d.get('fp32_verify') or {}).get('value'), (d.get('fp32_verify') or {}).get('max_abs_vs_bf16'))" 2>&1 | tail -1; done
python -c "
import json; d=json.load(open('$O/bench_cfg3_sustained.json')); print('sustained', d['value'], d['clocks'], d['e2e']['value'])"
head -c 400 $O/ref_cfg3.json
tail -2 $O/ncu_full.log
timeout 600 python tools/serve_bench.py --workload cfg3 --gpus 1 --requests 8000 --window 128 --frame 64 > $O/serve_cfg3.log 2>&1
tail -1 $O/serve_cfg3.log | cut -c1-300
