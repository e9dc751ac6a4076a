#!/bin/bash
# recall@10 vs T on cfg3 for both noise readings (developer tool; the labelled sensitivity runs of DESIGN.md §4)
mkdir -p gpurun_out/sweep
for noise in per_coord total; do
  for T in 500 2000 8000; do
    timeout 900 python bench.py --steps 3 --warmup 1 --T $T --noise $noise --no-cpu-baseline --no-e2e --recall-queries 200 \
      > gpurun_out/sweep/${noise}_T$T.log 2>&1
    tail -1 gpurun_out/sweep/${noise}_T$T.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$noise', $T, j['value'], j['ms_per_step'], j['recall'])"
  done
done
