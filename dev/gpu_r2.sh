#!/bin/bash
# round-2 check of the fused path: GPU tests, smoke, cfg3 bench, launch list, ncu full capture
O=gpurun_out/r2a; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench.json
timeout 600 python tools/prof_step.py cfg3 2 5 > $O/prof_step.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 10 --csv \
  --log-file $O/launches_cfg3.csv python tools/prof_step.py cfg3 3 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:5flame -c 10 -o $O/prof_full_cfg3 -f python tools/prof_step.py cfg3 1 > $O/ncu_full.log 2>&1
tail -3 $O/pytest_gpu.log; tail -3 $O/smoke.log; cat $O/prof_step.log | tail -14
python - <<PY
import json; d=json.load(open("$O/bench.json"))
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"].get("request_p99_ms"))
print("roof", json.dumps(d["roofline"])[:600]); print("clocks", d.get("clocks"))
PY
