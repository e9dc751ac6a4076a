#!/bin/bash
# refine group-mode experiments (developer tool; not bench values)
A="--n 200000 --nq 2048 --steps 2 --warmup 1 --no-cpu-baseline --recall-queries 0 --no-e2e"
run() { echo "$1 :: $(env $1 timeout 300 python bench.py $A 2>&1 | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["stages_ms"]["ms_refine"], j["fixup_sets_per_step"])')"; }
run "BVSS_REFINE_GROUP=0"
run "BVSS_REFINE_GROUP=1"
run "BVSS_REFINE_GROUP=1 BVSS_REFINE_RANGE=200000"
run "BVSS_REFINE_GROUP=1 BVSS_REFINE_RANGE=20000"
run "BVSS_REFINE_GROUP=1 BVSS_REFINE_QBLOCK=4"
