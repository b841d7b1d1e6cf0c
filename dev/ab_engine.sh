#!/bin/bash
# A/B of the host staging (engine.py) on one box: bench e2e with the current and dev/engine_prev.py
cp paper_2509_22681_b200/engine.py /tmp/engine_new.py
for rep in 1 2; do
  for v in new prev; do
    if [ $v = prev ]; then cp dev/engine_prev.py paper_2509_22681_b200/engine.py; else cp /tmp/engine_new.py paper_2509_22681_b200/engine.py; fi
    for w in ${WL:-cfg4 cfg1}; do
      timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2))"
    done
  done
done
cp /tmp/engine_new.py paper_2509_22681_b200/engine.py
