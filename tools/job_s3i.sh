# same-box A/B: in-tree (3 epilogue warps per lane quarter) vs B4 (4 per quarter, 96 registers, 228 B spills)
O=gpurun_out/s3i; mkdir -p $O
A="--steps 3 --warmup 3 --no-sweep --no-cpu-baseline --recall-queries 0 --no-e2e"
one() {
  local L=$1 P=$2; shift 2
  env BVSS_LIB=$P "$@" timeout 600 python bench.py $A 2>&1 | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('$L', '$*', 'refine_ms', round(j['stages_ms']['ms_refine'], 1), 'qps', j['value'], 'mhz', j['clocks']['sm_mhz'], 'surv', j['dense']['survivors_per_step'])"
}
{
for r in 1 2; do
one new ""
one B4 $PWD/tools/old_lib/B4/libbvss.so
done
} > $O/ab.log 2>&1
run() { echo "== $*"; env "$@" timeout 300 python tools/dense_smoke.py ${N:-1000000} ${NQ:-2000} 2>&1 | tail -1; }
{
run BVSS_LIB=
run BVSS_LIB=$PWD/tools/old_lib/B4/libbvss.so
run BVSS_LIB=$PWD/tools/old_lib/B4/libbvss.so BVSS_DENSE_DEBUG=1
run BVSS_LIB= BVSS_DENSE_DEBUG=1
} > $O/modes.log 2>&1
