#!/bin/bash
# emit-scan kernel time with and without the epilogue (developer tool)
CMD="bench.py --steps 1 --warmup 0 --no-cpu-baseline --recall-queries 0 --no-e2e"
mkdir -p gpurun_out
for d in 0 1; do
  BVSS_SCAN_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:scan_tc -c 2 --csv --log-file gpurun_out/scan_dbg$d.csv python $CMD > /dev/null 2>&1
  echo "dbg=$d"; grep scan_tc gpurun_out/scan_dbg$d.csv | python -c "
import csv,sys
for r in csv.reader(sys.stdin): print(r[4][:40], r[-3], r[-2], r[-1])"
done
