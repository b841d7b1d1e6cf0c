#!/bin/bash
# feature cache + dispatcher on the device, served-stream bench, cfg3 bench line
O=gpurun_out/r2b; mkdir -p $O
timeout 600 python -m pytest tests/test_service_cache_gpu.py tests/test_dispatch_gpu.py -q -x > $O/t.log 2>&1; echo rc=$? >> $O/t.log
tail -20 $O/t.log
timeout 900 python tools/serve_bench.py --workload cfg3 --gpus 1 --requests 2000 --window 256 > $O/serve_cfg3.log 2>&1
tail -3 $O/serve_cfg3.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench.json
python - <<PY
import json; d=json.load(open("$O/bench.json"))
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"].get("request_p99_ms"))
print("roof", json.dumps(d["roofline"])[:400]); print("cpu", json.dumps(d.get("cpu_baseline"))[:400])
PY
