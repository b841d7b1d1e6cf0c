#!/bin/bash
O=gpurun_out/r2e; mkdir -p $O
timeout 600 python -m pytest tests/test_dispatch_gpu.py -q -x > $O/t.log 2>&1; echo rc=$? >> $O/t.log; tail -3 $O/t.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench.json
python - <<PY
import json; d=json.load(open("$O/bench.json"))
r=d["roofline"]; print("value", d["value"], "e2e", d["e2e"]["value"], "frac", r["frac"], r["avg_launch_ms"], "hot", json.dumps(r.get("hot"))[:300])
PY
for fr in 16 64; do for w in 128 512; do
timeout 600 python tools/serve_bench.py --workload cfg3 --gpus 1 --requests 8000 --window $w --frame $fr > $O/serve_f${fr}_w$w.log 2>&1
tail -1 $O/serve_f${fr}_w$w.log | cut -c1-330
done; done
