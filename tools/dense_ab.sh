#!/bin/bash
# developer: dense brute force (1M sets x NQ queries), in-tree build vs tools/old_lib/head, alternating on one box
for r in 1 2; do
  echo "== old"; BVSS_LIB=$PWD/tools/old_lib/head/libbvss.so timeout 300 python tools/dense_smoke.py ${N:-1000000} ${NQ:-2000} 2>&1 | tail -1
  echo "== new"; timeout 300 python tools/dense_smoke.py ${N:-1000000} ${NQ:-2000} 2>&1 | tail -1
done
