#!/bin/bash
# interleaved A/B of env settings on the graph-replay step: dev/step_ab.sh WORKLOAD ROUNDS "ENV_A" "ENV_B" ...
w=$1; n=$2; shift 2
for r in $(seq $n); do
  for e in "$@"; do
    env $e python dev/step_time.py $w "$e" 2>&1 | tail -1
  done
done
