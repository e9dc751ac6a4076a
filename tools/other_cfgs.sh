#!/bin/bash
# the other BASELINE configs at scale on one GPU (developer tool)
mkdir -p gpurun_out/cfgs
for c in cfg2 cfg4 cfg1; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --recall-queries 50 > gpurun_out/cfgs/$c.log 2>&1
  tail -1 gpurun_out/cfgs/$c.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$c', j['value'], j['ms_per_step'], j['stages_ms'], j['recall'], j['select'], j['build'])" || tail -5 gpurun_out/cfgs/$c.log
done
