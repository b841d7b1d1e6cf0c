#!/bin/bash
# quick GPU iteration: parity tests + eager per-kernel profile of cfg3
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python tools/prof_step.py ${1:-cfg3} 2 7
