# full GPU suite (lane-per-vector encoder, dyn dense, group), encoder A/B, range sizes, bench
O=gpurun_out/s3d; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python tools/enc_ab.py cfg3 200000 > $O/enc_ab.log 2>&1
timeout 300 python tools/enc_ab.py cfg4 50000 >> $O/enc_ab.log 2>&1
timeout 300 python tools/enc_ab.py cfg1 1000 >> $O/enc_ab.log 2>&1
run() { echo "== $*"; env "$@" timeout 300 python tools/dense_smoke.py ${N:-1000000} ${NQ:-2000} 2>&1 | tail -1; }
{
run BVSS_DENSE_TPR=512
run BVSS_DENSE_TPR=1024
run BVSS_DENSE_TPR=2048
} > $O/modes.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
