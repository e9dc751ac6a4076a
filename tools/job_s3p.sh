# static set split (in-tree) correctness + bench; A/B vs V64 (union refresh every 64 tiles instead of 32)
O=gpurun_out/s3p; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_group.py tests/test_gpu_scale.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
A="--steps 3 --warmup 3 --no-sweep --no-cpu-baseline --recall-queries 0 --no-e2e"
one() {
  local L=$1 P=$2; shift 2
  env BVSS_LIB=$P "$@" timeout 600 python bench.py $A 2>&1 | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('$L', '$*', 'refine_ms', round(j['stages_ms']['ms_refine'], 1), 'qps', j['value'], 'mhz', j['clocks']['sm_mhz'], 'surv', j['dense']['survivors_per_step'])"
}
{
for r in 1 2; do
one new ""
one V64 $PWD/tools/old_lib/V64/libbvss.so
done
} > $O/ab.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
