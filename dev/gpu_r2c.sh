#!/bin/bash
# cache + dispatcher tests, full GPU suite, bench line (gated profile pass), served-stream bench
O=gpurun_out/r2c; mkdir -p $O
timeout 600 python -m pytest tests/test_service_cache_gpu.py tests/test_dispatch_gpu.py -q -x > $O/t.log 2>&1; echo rc=$? >> $O/t.log
tail -5 $O/t.log
timeout 900 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo rc=$? >> $O/all.log
tail -3 $O/all.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench.json
python - <<PY
import json; d=json.load(open("$O/bench.json"))
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"].get("request_p99_ms"))
print("roof", json.dumps(d["roofline"])[:300])
for k,v in d["kernels"].items(): print(k, v)
PY
for w in 64 128; do
timeout 900 python tools/serve_bench.py --workload cfg3 --gpus 1 --requests 6000 --window $w > $O/serve_cfg3_w$w.log 2>&1
tail -1 $O/serve_cfg3_w$w.log
done
