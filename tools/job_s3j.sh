# same-box A/B: P0 (one set per TMEM read) vs in-tree (adjacent set pairs read as one run)
O=gpurun_out/s3j; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_group.py tests/test_gpu_scale.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
A="--steps 3 --warmup 3 --no-sweep --no-cpu-baseline --recall-queries 0 --no-e2e"
one() {
  local L=$1 P=$2; shift 2
  env BVSS_LIB=$P "$@" timeout 600 python bench.py $A 2>&1 | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('$L', '$*', 'refine_ms', round(j['stages_ms']['ms_refine'], 1), 'qps', j['value'], 'mhz', j['clocks']['sm_mhz'], 'surv', j['dense']['survivors_per_step'])"
}
{
for r in 1 2; do
one P0 $PWD/tools/old_lib/P0/libbvss.so
one new ""
done
} > $O/ab.log 2>&1
run() { echo "== $*"; env "$@" timeout 300 python tools/dense_smoke.py ${N:-1000000} ${NQ:-2000} 2>&1 | tail -1; }
{
run BVSS_LIB=$PWD/tools/old_lib/P0/libbvss.so
run BVSS_LIB=
run BVSS_LIB= BVSS_DENSE_DEBUG=3
run BVSS_LIB= BVSS_DENSE_DEBUG=1
NQ=500 N=200000 run BVSS_LIB=$PWD/tools/old_lib/P0/libbvss.so
NQ=500 N=200000 run BVSS_LIB=
} > $O/modes.log 2>&1
