# dense kernel: union refresh period / stagger with the lane-rank k-th (developer tool)
O=gpurun_out/s4f; mkdir -p $O
timeout 900 python tools/dense_env_ab.py 1000000 2000 "" "BVSS_DENSE_REFRESH=16,4" "BVSS_DENSE_REFRESH=8,2" \
  "BVSS_DENSE_REFRESH=64,8" "BVSS_DENSE_REFRESH=32,0" "BVSS_DENSE_REFRESH=32,11" > $O/ab.log 2>&1; echo "rc=$?" >> $O/ab.log
