#!/bin/bash
# round measurement: parity tests, smoke, parity report, bench lines for every workload,
# the reference (CPU) arm, ncu launch list + full capture of one cfg3 pass
O=gpurun_out/measure; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/smoke.log
timeout 600 python tools/parity_report.py --json $O/parity.json > $O/parity.log 2>&1
for w in cfg3 cfg4 cfg2 cfg5 cfg1 cfg3_l2; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > $O/bench_$w.log 2>&1
  tail -1 $O/bench_$w.log > $O/bench_$w.json
done
# sustained: 150 back-to-back steps (the power cap shows after ~0.1 s of full load)
timeout 900 python bench.py --workload cfg3 --steps 150 --warmup 5 --no-cpu-baseline > $O/bench_cfg3_sustained.log 2>&1
tail -1 $O/bench_cfg3_sustained.log > $O/bench_cfg3_sustained.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_cfg3.log 2>&1; tail -1 $O/ref_cfg3.log > $O/ref_cfg3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 10 --csv \
  --log-file $O/launches_cfg3.csv python tools/prof_step.py cfg3 3 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:5flame -c 10 -o $O/prof_full_cfg3 -f python tools/prof_step.py cfg3 1 > $O/ncu_full.log 2>&1
tail -2 $O/pytest_gpu.log; tail -2 $O/smoke.log
for w in cfg3 cfg4 cfg2 cfg5 cfg1; do python -c "
import json; d=json.load(open('$O/bench_$w.json')); print('$w', round(d['value']/1e6,3), 'M/s e2e', round(d['e2e']['value']/1e6,3), 'p99', round(d['p99_ms'],2), 'roof', d['roofline']['kernel'], d['roofline']['frac'], 'cpu', (d.get('cpu_baseline') or {}).get('value'))" 2>&1 | tail -1; done
cat $O/ref_cfg3.json | head -c 300
