#!/bin/bash
# A/B of library builds on the cfg3 bench (developer tool; not bench values): every
# libbvss.so under tools/old_lib/ (older builds) and the in-tree build, alternating, ROUNDS times
A="--steps 3 --warmup 2 --no-cpu-baseline --recall-queries 0 --no-e2e"
LIBS="$(find tools/old_lib -name libbvss.so | sort) new"
for r in $(seq ${ROUNDS:-2}); do
  for L in $LIBS; do
    if [ $L = new ]; then P=""; else P=$PWD/$L; fi
    BVSS_LIB=$P python bench.py $A 2>&1 | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('$L', round(j['stages_ms']['ms_refine'], 2), j['stages_ms'], j['clocks']['sm_mhz'], j.get('build', {}).get('ms'))"
  done
done
