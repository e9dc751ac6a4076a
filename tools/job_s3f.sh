# candidate bitmap prefetched per tile + early exit of the survivor column scan; dense/scale/group tests; bench
O=gpurun_out/s3f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_scale.py tests/test_gpu_group.py tests/test_gpu_dist.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
run() { echo "== $*"; env "$@" timeout 300 python tools/dense_smoke.py ${N:-1000000} ${NQ:-2000} 2>&1 | tail -1; }
{
run BVSS_DENSE_LD=1
run BVSS_DENSE_LD=0
run BVSS_DENSE_DEBUG=3
run BVSS_DENSE_DEBUG=1
} > $O/modes.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
