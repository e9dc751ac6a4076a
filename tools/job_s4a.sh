# round-2 session 4: full-size parity, one-rank NCCL sharded search, launch list + ncu --set full of the dense
# kernel at HEAD (each ncu pass only after its command exited 0 without ncu)
O=gpurun_out/s4a; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_dist.py -x -q -rA > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
CMD="bench.py --steps 2 --warmup 3 --no-sweep --recall-queries 200 --no-cpu-baseline --no-e2e"
KR='regex:scan|select|refine|topk|encode|flyhash|sketch|expand|gather_sample|merge|pad_rows|max_float|dense|gate|alg2|fill'
timeout 900 python $CMD > $O/plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -c 3000 --csv --log-file $O/launches.csv \
  python $CMD > $O/ncu_launch.log 2>&1; echo "rc=$?" >> $O/ncu_launch.log
CMD1="tools/dense_smoke.py 1000000 2000"
timeout 300 python $CMD1 > $O/plain1.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dense_hausdorff -c 1 \
  -o $O/dense_full python $CMD1 > $O/ncu_full.log 2>&1; echo "rc=$?" >> $O/ncu_full.log
