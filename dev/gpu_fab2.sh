#!/bin/bash
mkdir -p gpurun_out/fab
FLAME_FUSED_ATTN=0 timeout 120 python dev/fused_ab.py gpurun_out/fab/unfused.npz
FLAME_FUSED_ATTN=1 timeout 120 python dev/fused_ab.py gpurun_out/fab/fused.npz
python -c "
import numpy as np
a=np.load('gpurun_out/fab/unfused.npz'); b=np.load('gpurun_out/fab/fused.npz')
for k in a.files: print(k, float(np.abs(a[k]-b[k]).max()))"
timeout 300 python -m pytest tests/test_forward_gpu.py -q -x > gpurun_out/fab/t.log 2>&1; echo rc=$?; tail -2 gpurun_out/fab/t.log
for m in 1 0; do for w in cfg5 cfg3; do FLAME_FUSED_ATTN=$m timeout 300 python tools/prof_step.py $w 2 5 > gpurun_out/fab/p_${w}_$m.log 2>&1; echo "$w mode $m"; grep -E "attention|qkv_cand|sum" gpurun_out/fab/p_${w}_$m.log; done; done
