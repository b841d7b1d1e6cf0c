#!/bin/bash
# parity tests + interleaved A/B bench: A = default, B = env override in $1 (A B A B)
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
fi
summ() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value']/1e6,3),'M ms',round(d['ms_per_step'],4),'e2e',round(d['e2e']['value']/1e6,3), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])
for k,v in d['kernels'].items(): print(f'  {k:18s} {v[\"ms_per_step\"]:.4f} {v[\"tflops\"]} {v[\"gbs\"]}')" | head -${2:-20}; }
for rep in 1 2; do
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_a$rep.log 2>&1; echo "== A$rep"; summ gpurun_out/bench_a$rep.log
[ -z "$1" ] && break
env $1 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_b$rep.log 2>&1; echo "== B$rep $1"; summ gpurun_out/bench_b$rep.log
done
