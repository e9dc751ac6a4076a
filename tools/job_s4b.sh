# dense kernel: union-refresh period / stagger and the lane-rank union k-th, A/B in one process (developer tool)
O=gpurun_out/s4b; mkdir -p $O
timeout 900 python tools/dense_env_ab.py 1000000 2000 "BVSS_DENSE_UKTH=0" "" "BVSS_DENSE_REFRESH=64,8" \
  "BVSS_DENSE_REFRESH=32,0" "BVSS_DENSE_REFRESH=128,8" "BVSS_DENSE_REFRESH=16,4" > $O/ab.log 2>&1; echo "rc=$?" >> $O/ab.log
