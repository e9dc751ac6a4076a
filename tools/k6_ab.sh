#!/bin/bash
# A/B of the packed K6 variants (BVSS_K6_VARIANT: 1 = 16 rows x 8 float4, 2 = 8 x 8, 0 = 8 x 4 at 3 CTAs/SM)
# on the T=2000 configuration: prints the fix-up stage time of each.
for v in 1 2 0 1 2 0; do
  BVSS_K6_VARIANT=$v timeout 400 python bench.py --T 2000 --no-sweep --steps 3 --warmup 3 --recall-queries 0 \
    --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('variant $v', d['stages_ms']['ms_topk'], d['clocks']['sm_mhz'])"
done
