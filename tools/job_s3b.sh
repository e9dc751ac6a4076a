# dense kernel A/B: dynamic range-major units (BVSS_DENSE_DYN) x exact-width TMEM loads (BVSS_DENSE_LD)
O=gpurun_out/s3b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_scale.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
run() { echo "== $*"; env "$@" timeout 300 python tools/dense_smoke.py ${N:-1000000} ${NQ:-2000} 2>&1 | tail -1; }
{
for rep in 1 2; do
run BVSS_DENSE_DYN=0 BVSS_DENSE_LD=0
run BVSS_DENSE_DYN=1 BVSS_DENSE_LD=0
run BVSS_DENSE_DYN=0 BVSS_DENSE_LD=1
run BVSS_DENSE_DYN=1 BVSS_DENSE_LD=1
done
run BVSS_DENSE_DYN=1 BVSS_DENSE_LD=1 BVSS_DENSE_TPR=64
run BVSS_DENSE_DYN=1 BVSS_DENSE_LD=1 BVSS_DENSE_TPR=256
run BVSS_DENSE_DYN=1 BVSS_DENSE_LD=1 BVSS_DENSE_DEBUG=1
run BVSS_DENSE_DYN=1 BVSS_DENSE_LD=1 BVSS_DENSE_DEBUG=4
run BVSS_DENSE_DYN=0 BVSS_DENSE_LD=1 BVSS_DENSE_DEBUG=1
NQ=10000 run BVSS_DENSE_DYN=0 BVSS_DENSE_LD=0
NQ=10000 run BVSS_DENSE_DYN=1 BVSS_DENSE_LD=1
} > $O/modes.log 2>&1
