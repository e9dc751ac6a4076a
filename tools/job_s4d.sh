# dense kernel: producer L2 prefetch of tile t + ahead (ahead,mod), A/B in one process (developer tool)
O=gpurun_out/s4d; mkdir -p $O
timeout 900 python tools/dense_env_ab.py 1000000 2000 "" "BVSS_DENSE_L2PF=4,8" "BVSS_DENSE_L2PF=8,8" \
  "BVSS_DENSE_L2PF=8,32" "BVSS_DENSE_L2PF=16,32" "BVSS_DENSE_L2PF=4,1" > $O/ab.log 2>&1; echo "rc=$?" >> $O/ab.log
