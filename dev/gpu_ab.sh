#!/bin/bash
# parity tests + bench; then bench again with the env override in $1 (A/B)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
summ() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value']/1e6,3),'M ms',round(d['ms_per_step'],4),'e2e',round(d['e2e']['value']/1e6,3), 'clk', d['clocks']['sm_mhz'])
for k,v in d['kernels'].items(): print(f'  {k:18s} {v[\"ms_per_step\"]:.4f} {v[\"tflops\"]} {v[\"gbs\"]}')"; }
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_a.log 2>&1; echo "== A"; summ gpurun_out/bench_a.log
if [ -n "$1" ]; then env $1 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_b.log 2>&1; echo "== B $1"; summ gpurun_out/bench_b.log; fi
