#!/bin/bash
# timing experiments on the refine kernel (developer tool; results are not bench values)
A="--steps 3 --warmup 1 --no-cpu-baseline --recall-queries 0 --no-e2e"
for e in ${EXPS:-0 1 2 3}; do
  BVSS_REFINE_EXPERIMENT=$e python bench.py $A 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('experiment', $e, j['stages_ms'])"
done
