#!/bin/bash
# scan kernel ablation (developer tool; results are not bench values)
for d in 0 1 2 4 3 7; do
  echo "dbg=$d $(BVSS_SCAN_DBG=$d timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --recall-queries 0 --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["stages_ms"]["ms_scan"], j["select"])')"
done
