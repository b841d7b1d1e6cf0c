#!/bin/bash
# fused-attention bring-up: parity tests (bounded), then the per-kernel profile and a bench line
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_forward_gpu.py -x -q > gpurun_out/fx_forward.log 2>&1; echo rc=$? >> gpurun_out/fx_forward.log
tail -15 gpurun_out/fx_forward.log
timeout 300 python -m pytest tests/test_parity_r2_gpu.py tests/test_dso_gpu.py tests/test_pda_gpu.py -x -q > gpurun_out/fx_more.log 2>&1; echo rc=$? >> gpurun_out/fx_more.log
tail -5 gpurun_out/fx_more.log
timeout 300 python tools/prof_step.py cfg3 2 5
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/fx_bench.log 2>&1
tail -1 gpurun_out/fx_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'])
for k,v in d['kernels'].items(): print(k, v)"
