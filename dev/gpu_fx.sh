#!/bin/bash
# fused-attention change: parity, per-kernel timing, trace
O=gpurun_out/fx; mkdir -p $O
timeout 600 python -m pytest tests/test_forward_gpu.py tests/test_parity_r2_gpu.py tests/test_dso_gpu.py -q -x > $O/t.log 2>&1; echo rc=$? >> $O/t.log
tail -4 $O/t.log
timeout 300 python tools/prof_step.py cfg3 2 5 > $O/prof.log 2>&1; tail -11 $O/prof.log
FLAME_B200_LIB=dev/var_trace.so timeout 300 python dev/fattn_trace.py cfg3 > $O/trace.log 2>&1; grep -A12 "^slot [02]" $O/trace.log | grep -v "@"
