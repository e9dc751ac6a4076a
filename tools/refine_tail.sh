#!/bin/bash
# refine gather variants on cfg3 (developer tool; results are not bench values):
# VARIANTS = comma-separated "TAIL KCS" pairs; TAIL=1 reads only the m real rows of every set
A="--steps 3 --warmup 2 --no-cpu-baseline --recall-queries 0 --no-e2e"
IFS=',' read -ra VS <<< "${VARIANTS:-0 2,1 2,1 1,0 1,1 3}"
for v in "${VS[@]}"; do
  set -- $v
  BVSS_REFINE_TAIL=$1 BVSS_REFINE_KCS=$2 python bench.py $A 2>&1 | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('tail', $1, 'kcs', $2, j['value'], j['stages_ms'], j.get('clocks'))"
done
