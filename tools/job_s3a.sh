O=gpurun_out/s3a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
for dbg in 0 1 2 4 0; do echo "== debug $dbg"; BVSS_DENSE_DEBUG=$dbg timeout 300 python tools/dense_smoke.py 1000000 2000 2>&1 | tail -1; done > $O/modes.log 2>&1
