#!/bin/bash
# ncu --set full of one eager pass, default and with the env override in $1
W=${W:-cfg3}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:${KREGEX:-5flame} -s ${NS:-0} -c ${NK:-11} -o gpurun_out/prof_a -f python tools/prof_step.py $W 1 > gpurun_out/ncu_a.log 2>&1
if [ -n "$1" ]; then env $1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:${KREGEX:-5flame} -s ${NS:-0} -c ${NK:-11} -o gpurun_out/prof_b -f python tools/prof_step.py $W 1 > gpurun_out/ncu_b.log 2>&1; fi
tail -2 gpurun_out/ncu_a.log
