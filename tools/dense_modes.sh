#!/bin/bash
# dense kernel: full / MMA-only (1) / no-survivor epilogue (3), alternating on one box (developer tool)
for r in 1 2; do for dbg in ${DBGS:-0 1 3}; do echo "== debug $dbg"; BVSS_DENSE_DEBUG=$dbg timeout 300 python tools/dense_smoke.py ${N:-1000000} ${NQ:-2000} 2>&1 | tail -1; done; done
