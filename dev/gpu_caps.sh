#!/bin/bash
O=gpurun_out/caps; mkdir -p $O
timeout 600 python -m pytest tests/test_caps_gpu.py tests/test_ops_gpu.py -q -x > $O/t.log 2>&1; echo rc=$? >> $O/t.log
tail -25 $O/t.log
timeout 900 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo rc=$? >> $O/all.log
tail -3 $O/all.log
