#!/bin/bash
# A/B of library builds on the dense brute force (developer tool): every tools/old_lib/*/libbvss.so and the
# in-tree build, alternating, ROUNDS times, on one box (box-to-box clock spread is +-20% for this kernel)
N=${N:-1000000}; NQ=${NQ:-2000}
LIBS="$(find tools/old_lib -name libbvss.so | sort) new"
for r in $(seq ${ROUNDS:-2}); do
  for L in $LIBS; do
    if [ $L = new ]; then P=""; else P=$PWD/$L; fi
    echo "== $L"; BVSS_LIB=$P timeout 300 python tools/dense_smoke.py $N $NQ 2>&1 | tail -1
  done
done
