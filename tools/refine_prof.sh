#!/bin/bash
# per-role wait breakdown of the refine kernel (developer tool)
A="--n ${N:-200000} --nq 2048 --steps 1 --warmup 0 --no-cpu-baseline --recall-queries 0 --no-e2e"
for g in ${GROUPS_:-0 1}; do
  echo "== group $g"
  BVSS_REFINE_PROF=1 BVSS_REFINE_GROUP=$g python bench.py $A 2>&1 | grep "refine prof" | tail -2
done
