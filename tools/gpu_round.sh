#!/bin/bash
# Round evidence pass (developer tool): GPU tests, smoke, default bench, launch list, ncu --set full of the
# dominant kernel on the default workload.  Results under gpurun_out/round/.
O=gpurun_out/round; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
CMD="bench.py --steps 2 --warmup 1 --no-cpu-baseline --recall-queries 0 --no-e2e"
KR='regex:scan|select|refine|topk|encode|flyhash|sketch|expand|gather_sample|merge|pad_rows|max_float'
python $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -c 2000 --csv --log-file $O/launches.csv \
  python $CMD > $O/ncu_launch.log 2>&1; echo "rc=$?" >> $O/ncu_launch.log
CMD1="bench.py --steps 1 --warmup 0 --no-cpu-baseline --recall-queries 0 --no-e2e"
python $CMD1 > $O/plain1.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:${PK:-refine_tc|scan_tc|topk_exact}" -s ${PS:-0} -c ${PC:-4} \
  -o $O/full python $CMD1 > $O/ncu_full.log 2>&1; echo "rc=$?" >> $O/ncu_full.log
