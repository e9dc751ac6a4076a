#!/bin/bash
# Round-2 final evidence (developer tool): launch list of the bench step, ncu --set full of ONE timed-step
# dense launch (the bench's own configuration: 10k queries, T = 600k, candidate bitmap), the dense kernel's
# per-role wait counters.  Each ncu command runs only after the same command exited 0 without ncu.
O=gpurun_out/r02s3; mkdir -p $O
CMD="bench.py --steps 2 --warmup 3 --no-sweep --recall-queries 0 --no-cpu-baseline --no-e2e"
KR='regex:scan|select|refine|topk|encode|flyhash|sketch|expand|gather_sample|merge|pad_rows|max_float|dense|gate|alg2|fill'
timeout 900 python $CMD > $O/plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -c 3000 --csv --log-file $O/launches.csv \
  python $CMD > $O/ncu_launch.log 2>&1; echo "rc=$?" >> $O/ncu_launch.log
CMD1="bench.py --steps 1 --warmup 3 --no-sweep --recall-queries 0 --no-cpu-baseline --no-e2e"
timeout 900 python $CMD1 > $O/plain1.log 2>&1 && \
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:dense_hausdorff -s 3 -c 1 \
  -o $O/dense_full python $CMD1 > $O/ncu_full.log 2>&1; echo "rc=$?" >> $O/ncu_full.log
BVSS_DENSE_PROF=1 timeout 300 python tools/dense_smoke.py 1000000 2000 > $O/dense_prof.log 2>&1
