# dense kernel at the session-4 default: sides timed apart (BVSS_DENSE_DEBUG 1/3/4) and per-role wait counters
O=gpurun_out/s4e; mkdir -p $O
timeout 900 python tools/dense_env_ab.py 1000000 2000 "" "BVSS_DENSE_DEBUG=1" "BVSS_DENSE_DEBUG=3" "BVSS_DENSE_DEBUG=4" \
  "BVSS_DENSE_PROF=1" > $O/modes.log 2>&1; echo "rc=$?" >> $O/modes.log
