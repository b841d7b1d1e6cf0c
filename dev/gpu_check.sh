#!/bin/bash
# one GPU round trip: parity tests, smoke, bench (used via gpurun)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'])
for k,v in d['kernels'].items(): print(f'{k:18s} {v[\"ms_per_step\"]:.4f} {v[\"tflops\"]} {v[\"gbs\"]}')"
