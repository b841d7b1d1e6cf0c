#!/bin/bash
# operator-level drop-in + plug-in tests, then the whole GPU suite
O=gpurun_out/ops; mkdir -p $O
timeout 600 python -m pytest tests/test_ops_gpu.py tests/test_plugin_gpu.py -q -x > $O/ops.log 2>&1; echo rc=$? >> $O/ops.log
tail -30 $O/ops.log
timeout 900 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo rc=$? >> $O/all.log
tail -5 $O/all.log
