# same-box A/B: in-tree (epilogue waits with a suspend-time hint) vs ST (static split of a tile's sets among the quarter's warps)
O=gpurun_out/s3o; mkdir -p $O
A="--steps 3 --warmup 3 --no-sweep --no-cpu-baseline --recall-queries 0 --no-e2e"
one() {
  local L=$1 P=$2; shift 2
  env BVSS_LIB=$P "$@" timeout 600 python bench.py $A 2>&1 | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('$L', '$*', 'refine_ms', round(j['stages_ms']['ms_refine'], 1), 'qps', j['value'], 'mhz', j['clocks']['sm_mhz'], 'encode_ms', j['stages_ms']['ms_encode'])"
}
{
for r in 1 2; do
one new ""
one ST $PWD/tools/old_lib/ST/libbvss.so
done
} > $O/ab.log 2>&1
