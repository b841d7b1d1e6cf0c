#!/bin/bash
# bench line + ncu full capture + launch list of the bench's own workload (tools/prof_step.py)
W=${1:-cfg3}
O=gpurun_out/bn_$W; mkdir -p $O
timeout 900 python bench.py --workload $W --steps 20 --warmup 5 > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench.json
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:5flame -c 12 -o $O/prof_full_$W -f python tools/prof_step.py $W 1 > $O/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 24 -c 12 --csv \
  --log-file $O/launches_$W.csv python tools/prof_step.py $W 3 > $O/ncu_launch.log 2>&1
python - <<PY
import json; d=json.load(open("$O/bench.json"))
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"].get("request_p99_ms"))
print("roof", json.dumps(d["roofline"])[:600])
for k,v in d["kernels"].items(): print(k, v)
print("pda", d.get("pda"))
PY
tail -3 $O/ncu_full.log
