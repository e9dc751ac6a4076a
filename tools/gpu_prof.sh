#!/bin/bash
# Profiling pass (developer tool): kernel launch list of the default bench (our kernels only),
# then ncu --set full on the top kernels of a medium run.  Each ncu command follows the same
# command run plainly (exit 0) as the profiling recipe requires.
mkdir -p gpurun_out
KR='regex:scan|select|refine|topk|encode|sketch|expand|gather_sample|merge|pad_rows|max_float'
if [ -z "$NOLAUNCH" ]; then
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --recall-queries 0 --no-e2e > gpurun_out/plain_full.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -c 2000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --recall-queries 0 --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/ncu_launch.log
fi
MED="bench.py --n 200000 --nq 2048 --steps 1 --warmup 0 --no-cpu-baseline --recall-queries 0 --no-e2e"
python $MED > gpurun_out/plain_med.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "${PK:-regex:scan_tc|refine_tc|topk_fixup}" -s ${PS:-0} -c ${PC:-3} \
  -o gpurun_out/prof python $MED > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
