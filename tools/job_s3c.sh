# dense kernel: running tau per query (dyn and static schedules), range sizes; group API tests
O=gpurun_out/s3c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_scale.py tests/test_gpu_group.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
run() { echo "== $*"; env "$@" timeout 300 python tools/dense_smoke.py ${N:-1000000} ${NQ:-2000} 2>&1 | tail -1; }
{
run BVSS_DENSE_DYN=0
run BVSS_DENSE_DYN=1 BVSS_DENSE_TPR=128
run BVSS_DENSE_DYN=1 BVSS_DENSE_TPR=256
run BVSS_DENSE_DYN=1 BVSS_DENSE_TPR=512
run BVSS_DENSE_DYN=0
run BVSS_DENSE_DYN=1 BVSS_DENSE_TPR=128
run BVSS_DENSE_DYN=1 BVSS_DENSE_TPR=256
run BVSS_DENSE_DYN=1 BVSS_DENSE_TPR=512
run BVSS_DENSE_DYN=1 BVSS_DENSE_TPR=256 BVSS_DENSE_DEBUG=3
run BVSS_DENSE_DYN=1 BVSS_DENSE_TPR=256 BVSS_DENSE_DEBUG=1
NQ=10000 run BVSS_DENSE_DYN=0
NQ=10000 run BVSS_DENSE_DYN=1 BVSS_DENSE_TPR=256
} > $O/modes.log 2>&1
