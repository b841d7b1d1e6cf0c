#!/bin/bash
# ncu --set full capture of one eager forward pass (11 kernels) of a workload
W=${1:-cfg3}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:5flame -c 11 -o gpurun_out/prof_full_$W -f python tools/prof_step.py $W 1 > gpurun_out/ncu_full_$W.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 22 -c 11 --csv \
  --log-file gpurun_out/launches_$W.csv python tools/prof_step.py $W 3 > gpurun_out/ncu_launch_$W.log 2>&1
tail -3 gpurun_out/ncu_full_$W.log
