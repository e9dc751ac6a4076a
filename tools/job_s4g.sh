# round-2 session-4 final evidence: GPU suite, smoke, bench, launch list + ncu --set full of one bench dense launch
O=gpurun_out/s4g; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
CMD="bench.py --steps 2 --warmup 3 --no-sweep --recall-queries 0 --no-cpu-baseline --no-e2e"
KR='regex:scan|select|refine|topk|encode|flyhash|sketch|expand|gather_sample|merge|pad_rows|max_float|dense|gate|alg2|fill'
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -c 3000 --csv --log-file $O/launches.csv \
  python $CMD > $O/ncu_launch.log 2>&1; echo "rc=$?" >> $O/ncu_launch.log
CMD1="bench.py --steps 1 --warmup 3 --no-sweep --recall-queries 0 --no-cpu-baseline --no-e2e"
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:dense_hausdorff -s 3 -c 1 \
  -o $O/dense_full python $CMD1 > $O/ncu_full.log 2>&1; echo "rc=$?" >> $O/ncu_full.log
