# same-box A/B: A = 06db916 (inheritance, N=240) vs the in-tree build (N=256, bitmap prefetch, early exit,
# other-k loads consumed a tile later); range sizes on the bench workload
O=gpurun_out/s3g; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_group.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
A="--steps 3 --warmup 3 --no-sweep --no-cpu-baseline --recall-queries 0 --no-e2e"
one() {  # label, lib, env...
  local L=$1 P=$2; shift 2
  env BVSS_LIB=$P "$@" timeout 600 python bench.py $A 2>&1 | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('$L', '$*', 'refine_ms', round(j['stages_ms']['ms_refine'], 1), 'qps', j['value'], 'mhz', j['clocks']['sm_mhz'], 'surv', j['dense']['survivors_per_step'])"
}
{
for r in 1 2; do
one A $PWD/tools/old_lib/A/libbvss.so
one new ""
done
one new "" BVSS_DENSE_TPR=128
one new "" BVSS_DENSE_TPR=256
one new "" BVSS_DENSE_TPR=512
one A $PWD/tools/old_lib/A/libbvss.so BVSS_DENSE_TPR=256
one new ""
} > $O/ab.log 2>&1
run() { echo "== $*"; env "$@" timeout 300 python tools/dense_smoke.py ${N:-1000000} ${NQ:-2000} 2>&1 | tail -1; }
{
run BVSS_LIB=$PWD/tools/old_lib/A/libbvss.so
run BVSS_LIB=
run BVSS_LIB= BVSS_DENSE_DEBUG=3
run BVSS_LIB= BVSS_DENSE_DEBUG=1
run BVSS_LIB= BVSS_DENSE_DEBUG=4
} > $O/modes.log 2>&1
