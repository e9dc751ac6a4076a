#!/bin/bash
# ncu --set full of the fused emit scan on the default cfg3 workload (developer tool)
mkdir -p gpurun_out
CMD="bench.py --steps 1 --warmup 0 --no-cpu-baseline --recall-queries 0 --no-e2e"
python $CMD > gpurun_out/plain_fs.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${PK:-scan_tc}" -s ${PS:-1} -c 1 \
  -o gpurun_out/prof_fs python $CMD > gpurun_out/ncu_fs.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_fs.log
