# full GPU suite; dense list inheritance at 512/1024/2048-tile ranges; bench
O=gpurun_out/s3e; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
run() { echo "== $*"; env "$@" timeout 300 python tools/dense_smoke.py ${N:-1000000} ${NQ:-2000} 2>&1 | tail -1; }
{
run BVSS_DENSE_TPR=512
run BVSS_DENSE_TPR=1024
run BVSS_DENSE_TPR=2048
run BVSS_DENSE_TPR=1024 BVSS_DENSE_DEBUG=3
NQ=500 run BVSS_DENSE_TPR=1024
NQ=500 run BVSS_DENSE_DYN=0
} > $O/modes.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
