#!/bin/bash
# dense kernel: the number of database ranges per query tile pair (developer tool), MMA-only and full
for r in 1 2; do for R in ${RS:-1 4 16}; do for dbg in ${DBGS:-1 0}; do echo "== R $R debug $dbg"; BVSS_DENSE_R=$R BVSS_DENSE_DEBUG=$dbg timeout 300 python tools/dense_smoke.py ${N:-1000000} ${NQ:-2000} 2>&1 | tail -1; done; done; done
