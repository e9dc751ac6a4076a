// dense.cu — K8d: candidate-major (dense) Hausdorff top-k on the 5th-generation
// tensor cores, with a rigorous branch-and-bound prune (Def 4; Alg 6
// lines 19-23 P:809-814; "precise calculations" for the brute force).
//
// When the candidate budget T is a large fraction of n (the recall@10 >= 0.9
// operating point of the synthetic workloads) or T = n (K8, the
// recall ground truth), gathering each query's candidates (K5, query-major)
// moves T x (set rows) x d x 2 bytes per query.  This kernel instead streams the
// database ONCE per 128-row query tile: the query tile is the stationary A
// operand (M = 128 packed query rows, resident in shared memory), the database
// rows stream through a TMA ring as the B operand (N = 256 rows per tile, K = d
// in 64-element SW128 chunks), and tcgen05.mma accumulates the Gram tile in TMEM
// (two 256-column accumulators, double-buffered against the epilogue).
//
// Layouts (built once per index / per batch):
//   database  hd [nvec][dpad] fp16 = x / S_db, one global power-of-two scale
//             S_db >= max|x| (row-major; tiles are runs of whole consecutive sets
//             of <= 256 rows, any start row: TMA swizzles on the fly);
//   queries   qd [ntq*128][dpad] fp16 = x / S_q, query sets packed into 32-row
//             warp bins (a set never straddles a warp), 4 bins per tile.
// The squared norm of every database row rides in the MMA as one extra K = 16
// chunk (SWIZZLE_32B): the database row carries (h, l) = the fp16 split of
// |v|^2 / S_db^2, the query row carries (alpha, alpha) with alpha = -S_db / (2 S_q)
// (powers of two, exact), so the accumulator is
//     acc(q, v) = sum_k (q_k / S_q)(v_k / S_db) + alpha (h + l)
// and D^2(q, v) = |q|^2 + kappa acc(q, v), kappa = -2 S_q S_db < 0.  Hence
// min_v D^2 = |q|^2 + kappa max_v acc: one FMNMX per accumulator value.
//
// Epilogue (12 warps, three per TMEM lane quarter; lane = query row, column =
// database row; sets of a tile alternate between the warps of a quarter):
//   per database set V and lane q:   r_q = max(0, |q|^2 + kappa max_v acc)  (lane-local)
//   A(Q, V) = max_{q in Q} r_q  is a lower bound of H^2(Q, V) = max(A, B).
// Branch and bound per query: tau_Q = the k-th smallest upper bound (H2c + E)
// among the sets seen so far (a list of k per (query, range, epilogue warp) in
// global memory; any k distinct sets' upper bounds bound the true k-th H^2).
// A set is pruned when some lane of Q has r_q > tau_Q + E (so A - E > tau_Q:
// its exact H^2 exceeds the exact k-th, the set cannot be in the top-k).  A set
// that survives gets B(Q, V) = max_v min_q D^2 by one redux.sync.min per column
// (TMEM re-read; survivors are rare once tau has settled), H2c = max(A, B), and
// is emitted to the query's candidate list when H2c - E <= tau_Q.  K6
// (topk_exact_kernel) then recomputes the final window exactly in fp32: the
// emitted lists contain every set whose H2c - E <= the final U_k, which is the
// K6 window rule, so the result is exact (E from error_consts()).
//
// CTA = 15 warps: 0 TMA producer, 1 TMEM owner + MMA issuer (one thread), 2-13
// epilogue, 14 tile info (set columns / sizes and column norms into shared memory).  Persistent: unit u = blockIdx.x + i * gridDim.x is (query tile
// u / R, database range u % R); consecutive units run the same ranges at the
// same time on all SMs, so each database tile is read from HBM about once per
// wave and served from L2 to the other CTAs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "tc.cuh"


namespace bvss {

// database rows per tile (MMA N): two 256-column accumulators fill the 512-column allocation; the epilogue's
// exact-width reads never pass a set's last column (a load past column 511 faults: tools/test_tmem_ld.cu), and
// sets start at any column (unaligned loads are legal).  A tcgen05.mma costs about the same for any N <= 256
// (tools/microbench_umma.cu), so the widest tile does the most work per instruction.
constexpr int kDenseN = 256;
constexpr int kDenseM = 128;      // packed query rows per tile (MMA M)
constexpr int kEpiSub = 3;                                  // epilogue warps per TMEM lane quarter
constexpr int kEpiWarpsD = 4 * kEpiSub;
constexpr int kInfoWarp = 2 + kEpiWarpsD;
constexpr int kDenseThreads = 32 * (kInfoWarp + 1);        // producer, MMA, epilogue, tile info
constexpr int kInfoSlotsD = 4;
constexpr int kDenseMaxStages = 8;
constexpr int kUnitQ = 4;          // published unit ids in flight (dyn scheduling)
// consumers of a published unit id: the peer's producer, the leader's MMA thread, both CTAs' info warps and
// epilogue warps
constexpr int kUnitConsumers = 1 + 1 + 2 + 2 * kEpiWarpsD;
constexpr uint32_t kAChunkBytes = kDenseM * 128;  // one 64-element K chunk of the query tile (16 KB)
// CTA pairs (cta_group::2): one tcgen05.mma M=256 N=256 per K step covers the two CTAs' query tiles (128
// rows each, A in each CTA's shared memory) against one database tile whose rows are split between the
// CTAs (120 each): every SM streams half of the tile, so the L2 -> SM traffic per flop halves
constexpr int kHalfN = kDenseN / 2;
constexpr uint32_t kBChunkBytes = kHalfN * 128;   // this CTA's half of one K chunk of a database tile (16 KB)
constexpr uint32_t kAAugBytes = kDenseM * 32;     // the query tile's norm chunk (K = 16 halves = 32 B rows)
constexpr uint32_t kBAugBytes = kHalfN * 32;      // this CTA's half of a database tile's norm chunk

// SWIZZLE_32B K-major descriptor (8-row atoms of 8 x 32 B, SBO = 256 B; layout type 6, version 1)
__device__ __forceinline__ uint64_t sw32_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>(256u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(6u) << 61;
  return d;
}

struct DenseArgs {
  CUtensorMap tmA;              // qd [ntq*128][dpad] fp16, box {64, 128}, SWIZZLE_128B
  CUtensorMap tmB;              // hd [nvec][dpad] fp16, box {64, 120}, SWIZZLE_128B
  CUtensorMap tmAa;             // qa [128][16] fp16 (alpha, alpha, 0...), box {16, 128}, SWIZZLE_32B
  CUtensorMap tmBa;             // va [nvec][16] fp16 (h, l, 0...), box {16, 120}, SWIZZLE_32B
  int KC;                       // dpad / 64
  int stages;
  int ntq;                      // query tiles
  int R;                        // database ranges
  int ntiles;                   // database tiles
  const int32_t* tile_s0;       // [ntiles] first set of each tile
  const int32_t* tile_s1;       // [ntiles] one past the last set
  const int64_t* off;           // [n+1]
  const int32_t* lane_qid;      // [ntq*128] query of each packed row, -1 = padding
  const float* lane_qn;         // [ntq*128] squared norm of each packed row
  const float* qE;              // [nq] squared-distance error bound of each query
  float* tau0;                  // [nq] running tau of each query: an upper bound on its k-th H^2 (+inf if none),
                                // lowered (atomicMin on the bits; every value is >= 0) by every warp whenever
                                // it refreshes its own tau, read when a unit starts: a unit of range r starts
                                // from the bound of every range run before it, not only from the union of the
                                // last few ranges' lists
  float kappa;                  // -2 S_q S_db
  int k;
  float* lists;                 // [nq][R][kEpiSub][k] sorted upper bounds, +inf-initialised
  int32_t* cnt;                 // [nq] emitted candidates (may exceed cap: overflow)
  int32_t* ids;                 // [nq][cap]
  float* vals;                  // [nq][cap] tensor-core H^2
  int cap;
  const uint32_t* mask;         // optional candidate bitmap, row q at mask + q * mask_stride (bit i = set i)
  int64_t mask_stride;          // words per query row (0: one row shared by every query)
  int mask_last_word;           // last word of a row the kernel may read ((last set of the last tile) / 32)
  int64_t id_base;
  unsigned long long* stat;     // [2]: survivors, emitted (may be null)
  unsigned long long* prof;     // developer per-role cycle counters (env BVSS_DENSE_PROF) or null
  int debug;                    // developer switch BVSS_DENSE_DEBUG: 1 = epilogue skips its work, 2 = no MMAs,
                                // 3 = no survivor work, 4 = no database loads and no epilogue (timing only)
  uint32_t refresh_mask;        // union refresh every refresh_mask + 1 tiles (a power of two; default 32) ...
  uint32_t refresh_stagger;     // ... at tile_ctr + stagger * sub (default 8; developer env BVSS_DENSE_REFRESH=p,s)
  int l2pf_ahead, l2pf_mod;     // producer L2 prefetch of tile t + ahead by the pairs with pair % mod == t % mod
                                // (0: off; developer env BVSS_DENSE_L2PF=ahead,mod)
  int ukth_fast;                // union k-th by lane ranks when the union has <= 32 values, 2: with the loads of
                                // up to 4 query segments issued together (env BVSS_DENSE_UKTH=0 / 1 / 2, default 2)
  int dyn;                      // 1: units handed out by a global counter in range-major order (see pair_unit)
  int* unit_ctr;                // [1] next unit (dyn), zeroed before the launch
  int* udone;                   // [nqp][R] (dyn): epilogue warps that finished unit (qp, r), zeroed before the
                                // launch; a unit whose predecessor range is complete (2 kEpiWarpsD) inherits its
                                // lists, so each warp's list holds its best k over every range run so far
};

// per-tile metadata the info warp stages for the epilogue (shared memory): the database sets of the tile
// (first set id, count, column and size of each)
struct DenseInfo {
  int s0, nsets, pad0, pad1;
  int16_t col0[kDenseN];
  int16_t mv[kDenseN];
};

struct DenseCtl {
  DenseInfo info[kInfoSlotsD];
  uint64_t info_full[kInfoSlotsD], info_empty[kInfoSlotsD];
  uint64_t full[kDenseMaxStages];
  uint64_t empty[kDenseMaxStages];
  uint64_t a_full, a_empty;
  uint64_t tfull[2], tempty[2];
  int unitq[kUnitQ];                                  // unit ids published by the leader's producer (dyn)
  uint64_t unit_full[kUnitQ], unit_empty[kUnitQ];
  uint32_t tmem_base;
};

__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of one tensor box (no shared memory, no barrier): pulls a database tile into L2 ahead of the
// pairs that will load it
__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
// the same TMA with the pair's completion barrier in the leader CTA (cta_group::2: the bytes of both CTAs'
// loads complete on the leader's barrier, whose MMA thread consumes both halves)
__device__ __forceinline__ void tma_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar_leader) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_leader)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// shared::cluster address of the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// relaxed: the accumulator hand-back needs no memory ordering (tcgen05.wait::ld has completed the TMEM reads,
// and the release form costs a GPU-scope MEMBAR per tile: ncu)
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void expect_tx_remote(uint32_t cluster_addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void arrive_release_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {  // acquire at cluster scope
  const uint32_t addr = smem_u32(bar);
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
}
// the pair's MMA (issued by the leader): D[both CTAs' TMEM] (+)= A[both CTAs' smem] * B[both halves]^T
__device__ __forceinline__ void umma_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on the barrier at this offset in both CTAs once the leader's prior MMAs are done
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// 32 lanes x 32 bit, 32 consecutive columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ float fmax3(float a, float b, float c) { return fmaxf(a, fmaxf(b, c)); }  // FMNMX3

// The columns of a run of mvc (1..31) database rows starting at TMEM address taddr, for this lane's query row,
// read by the loads of mvc's binary digits (x16, x8, x4, x2, x1 at consecutive column offsets): exactly the
// set's columns (a 32 + 8 column form read 40 columns for a set of 18 rows and needed 32 spare TMEM columns
// past the last accumulator).  Branches are warp-uniform (one set per warp).
struct SetColsX {
  uint32_t a16[16], a8[8], a4[4], a2[2], a1[1];
};
__device__ __forceinline__ void tmem_ldx4(uint32_t t, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(t)
               : "memory");
}
__device__ __forceinline__ void tmem_ldx2(uint32_t t, uint32_t (&r)[2]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(t) : "memory");
}
__device__ __forceinline__ void tmem_ldx1(uint32_t t, uint32_t (&r)[1]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(t) : "memory");
}
__device__ __forceinline__ void load_set(uint32_t taddr, int mvc, SetColsX& c) {
  if (mvc & 16) {
    tc::tmem_ld16(taddr, c.a16);
    taddr += 16;
  }
  if (mvc & 8) {
    tmem_ld8(taddr, c.a8);
    taddr += 8;
  }
  if (mvc & 4) {
    tmem_ldx4(taddr, c.a4);
    taddr += 4;
  }
  if (mvc & 2) {
    tmem_ldx2(taddr, c.a2);
    taddr += 2;
  }
  if (mvc & 1) tmem_ldx1(taddr, c.a1);
  tc::tmem_ld_wait();
}
__device__ __forceinline__ float set_max(const SetColsX& c, int mvc) {
  float m = __int_as_float(0xff800000);
  if (mvc & 16) {
#pragma unroll
    for (int j = 0; j < 16; j += 2) m = fmax3(m, __uint_as_float(c.a16[j]), __uint_as_float(c.a16[j + 1]));
  }
  if (mvc & 8) {
#pragma unroll
    for (int j = 0; j < 8; j += 2) m = fmax3(m, __uint_as_float(c.a8[j]), __uint_as_float(c.a8[j + 1]));
  }
  if (mvc & 4) m = fmax3(m, fmax3(__uint_as_float(c.a4[0]), __uint_as_float(c.a4[1]), __uint_as_float(c.a4[2])),
                         __uint_as_float(c.a4[3]));
  if (mvc & 2) m = fmax3(m, __uint_as_float(c.a2[0]), __uint_as_float(c.a2[1]));
  if (mvc & 1) m = fmaxf(m, __uint_as_float(c.a1[0]));
  return m;
}
// (lim: the caller only needs B while B <= lim -- a survivor with B > tau + E can be neither inserted nor
// emitted -- so the scan stops after the first group of columns that exceeds it; warp-uniform)
__device__ __forceinline__ float set_colmin_max(const SetColsX& c, int mvc, float kappa, float qn, bool inseg,
                                                float lim = 3.402823466e38f) {
  float B = 0.0f;
  auto col = [&](uint32_t x) {
    const float d2 = fmaxf(fmaf(kappa, __uint_as_float(x), qn), 0.0f);
    B = fmaxf(B, __uint_as_float(__reduce_min_sync(0xffffffffu, inseg ? __float_as_uint(d2) : 0xffffffffu)));
  };
  if (mvc & 16) {
#pragma unroll
    for (int j = 0; j < 8; ++j) col(c.a16[j]);
    if (B > lim) return B;
#pragma unroll
    for (int j = 8; j < 16; ++j) col(c.a16[j]);
    if (B > lim) return B;
  }
  if (mvc & 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) col(c.a8[j]);
    if (B > lim) return B;
  }
  if (mvc & 4) {
#pragma unroll
    for (int j = 0; j < 4; ++j) col(c.a4[j]);
  }
  if (mvc & 2) {
    col(c.a2[0]);
    col(c.a2[1]);
  }
  if (mvc & 1) col(c.a1[0]);
  return B;
}

__device__ __forceinline__ float vload_volatile(const float* p);

// k-th smallest value of the union of a query's bound lists over nr <= R distinct ranges (from range r on) x
// kEpiSub warps: any k distinct sets' upper bounds bound the exact k-th H^2 from above, so the union's k-th is
// a valid (and much tighter) tau.  The lists are read while their owners may be inserting (a lane-parallel
// shift): a torn read can show one value at two adjacent positions of a list, which would count one set twice
// and make the k-th too small (an invalid tau: observed as a wrong top-k with R = 1).  So a value equal to its
// predecessor in the same list counts as +inf (two sets with equal bounds then count once: conservative).
// Warp-wide radix select on the (non-negative) float bits.
// (dir = +1: ranges r, r+1, ...; dir = -1: r, r-1, ... -- the ranges the range-major schedule has already run)
// The k-th smallest (with multiplicity) of one value per lane (lanes past the union hold +inf), after the
// dedup rule of union_kth (a value equal to its predecessor in the same sorted list of k is a torn read of a
// list being shifted and counts once): each lane's rank by 32 independent shuffles.
__device__ __forceinline__ float ukth_rank(float x, int k, int lane) {
  const float prev = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane % k != 0 && prev == x) x = __int_as_float(0x7f800000);
  int rank = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float y = __shfl_sync(0xffffffffu, x, j);
    rank += (y < x || (y == x && j < lane)) ? 1 : 0;
  }
  const unsigned at = __ballot_sync(0xffffffffu, rank == k - 1);
  return __shfl_sync(0xffffffffu, x, __ffs(at) - 1);
}

__device__ float union_kth(const float* lq0 /* lists of (q, range 0) */, int R, int r, int nr, int k, int lane,
                           int dir, bool fast) {
  const int per_range = kEpiSub * k, total = nr * per_range;
  if (fast && total <= 32) {  // one value per lane: the k-th smallest by rank (32 independent shuffles instead
                              // of 31 dependent warp reductions; same value, ties counted with multiplicity)
    float x = __int_as_float(0x7f800000);
    if (lane < total) x = vload_volatile(lq0 + static_cast<int64_t>((r + R + dir * (lane / per_range)) % R) * per_range + lane % per_range);
    return ukth_rank(x, k, lane);
  }
  float v[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int x = lane + 32 * e;
    v[e] = __int_as_float(0x7f800000);
    if (x < total) v[e] = vload_volatile(lq0 + static_cast<int64_t>((r + R + dir * (x / per_range)) % R) * per_range + x % per_range);
  }
  float last = __int_as_float(0x7f800000);  // lane 31's value of the previous row of 32
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int x = lane + 32 * e;
    float prev = __shfl_up_sync(0xffffffffu, v[e], 1);
    if (lane == 0) prev = last;
    last = __shfl_sync(0xffffffffu, v[e], 31);
    if (x < total && x % k != 0 && prev == v[e]) v[e] = __int_as_float(0x7f800000);
  }
  uint32_t prefix = 0;
  for (int bit = 30; bit >= 0; --bit) {  // largest x with count(< x) < k: the k-th smallest
    const uint32_t cand = prefix | (1u << bit);
    int c = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) c += __float_as_uint(v[e]) < cand ? 1 : 0;
    c = __reduce_add_sync(0xffffffffu, c);
    if (c < k) prefix = cand;
  }
  return __uint_as_float(prefix);
}

__device__ __forceinline__ float vload_volatile(const float* p) {
  float v;
  asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p));  // (gpu scope: L2-coherent)
  return v;
}

// The i-th work unit of this CTA pair (-1: none left).  Static (dyn = 0): u = pair + i * npairs, units
// ordered (query tile pair, range) pair-major.  Dynamic (dyn = 1): the leader's producer takes the next unit
// of a global counter when it starts a unit and publishes it to both CTAs (a kUnitQ-deep queue in shared
// memory); units are ordered range-major, so all pairs work on the same one or two database ranges at any
// moment and a range is read from HBM about once while every query tile pair streams it from L2 (pairs that
// run faster simply take more units: no drift apart along the database).  Every consumer releases the slot
// (pair_unit_release) once it has read it.
__device__ __forceinline__ int pair_unit(const DenseArgs& a, DenseCtl& S, int i, int pair, int npairs, int units,
                                         bool publisher) {
  if (!a.dyn) {
    const int u = pair + i * npairs;
    return u < units ? u : -1;
  }
  const int slot = i % kUnitQ;
  const uint32_t ph = static_cast<uint32_t>(i / kUnitQ) & 1u;
  if (publisher) {
    mbar_wait_cluster(&S.unit_empty[slot], ph ^ 1u);
    int u = atomicAdd(a.unit_ctr, 1);
    if (u >= units) u = -1;
    *reinterpret_cast<volatile int*>(&S.unitq[slot]) = u;
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(map_to(&S.unitq[slot], 1)), "r"(u) : "memory");
    arrive_release_cluster(map_to(&S.unit_full[slot], 0));
    arrive_release_cluster(map_to(&S.unit_full[slot], 1));
    return u;
  }
  mbar_wait_cluster(&S.unit_full[slot], ph);
  return *reinterpret_cast<volatile int*>(&S.unitq[slot]);
}
__device__ __forceinline__ void pair_unit_release(const DenseArgs& a, DenseCtl& S, int i) {
  if (a.dyn) arrive_release_cluster(map_to(&S.unit_empty[i % kUnitQ], 0));
}
// (query tile pair, database range) of unit u
__device__ __forceinline__ void unit_coords(const DenseArgs& a, int u, int* qp, int* r) {
  const int nqp = a.ntq / 2;
  if (a.dyn) {
    *r = u / nqp;
    *qp = u - *r * nqp;
  } else {
    *qp = u / a.R;
    *r = u - *qp * a.R;
  }
}

__device__ __forceinline__ void range_tiles(int r, int R, int ntiles, int* t0, int* t1) {
  *t0 = static_cast<int>((static_cast<int64_t>(ntiles) * r) / R);
  *t1 = static_cast<int>((static_cast<int64_t>(ntiles) * (r + 1)) / R);
}

// developer instrumentation: cycles spent in `call` added to prof[slot] (one counter per role and wait)
#define DPROF(slot, call)                                                   \
  do {                                                                      \
    if (a.prof) {                                                           \
      const long long t0_ = clock64();                                      \
      call;                                                                 \
      if ((threadIdx.x & 31) == 0) atomicAdd(&a.prof[slot], (unsigned long long)(clock64() - t0_)); \
    } else {                                                                \
      call;                                                                 \
    }                                                                       \
  } while (0)

__global__ void __launch_bounds__(kDenseThreads, 1) dense_hausdorff_kernel(const __grid_constant__ DenseArgs a) {
  using Cols = SetColsX;
  constexpr int CH = 31;  // columns per TMEM read of a set
  extern __shared__ __align__(1024) uint8_t dsm_raw[];
  __shared__ DenseCtl S;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t a_s = smem_u32(base);                                  // KC x 16 KB query tile
  const uint32_t aa_s = a_s + static_cast<uint32_t>(a.KC) * kAChunkBytes;  // 4 KB norm chunk of the query tile
  const uint32_t ring_s = aa_s + kAAugBytes;                               // stages x 30 KB
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NST = a.stages;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&S.full[s], 1);
      tc::mbar_init(&S.empty[s], 1);
    }
    tc::mbar_init(&S.a_full, 1);
    tc::mbar_init(&S.a_empty, 1);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&S.tfull[b], 1);
      tc::mbar_init(&S.tempty[b], 2 * kEpiWarpsD);  // (the leader's: both CTAs' epilogue warps arrive)
    }
    for (int b = 0; b < kUnitQ; ++b) {
      tc::mbar_init(&S.unit_full[b], 1);
      tc::mbar_init(&S.unit_empty[b], kUnitConsumers);
    }
    for (int b = 0; b < kInfoSlotsD; ++b) {
      tc::mbar_init(&S.info_full[b], 1);
      tc::mbar_init(&S.info_empty[b], kEpiWarpsD);
    }
    tc::fence_mbar_init();
  }
  cluster_sync_all();  // the leader's barriers exist before the peer's loads and arrivals target them
  if (warp == 1) {     // the pair's TMEM (same columns in both CTAs), allocated by the same warp of each CTA
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&S.tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync_all();
  tc::fence_after_sync();
  const uint32_t tmem = S.tmem_base;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const int pair = static_cast<int>(cluster_id_x()), npairs = static_cast<int>(nclusters_x());
  const int units = (a.ntq / 2) * a.R;  // pair units: (query tile pair, database range); ntq is even
  const uint32_t full_l0 = map_to(&S.full[0], 0), a_full_l = map_to(&S.a_full, 0);
  const uint32_t tempty_l0 = map_to(&S.tempty[0], 0);
  const long long t_start = clock64();

  if (warp == 0) {
    // =========================== TMA producer (one thread per CTA) ===========================
    // each CTA loads its own query tile and its half of every database tile; the bytes of both CTAs complete
    // on the leader's barriers, armed (expect_tx of the pair's bytes) by the leader's producer
    if (lane == 0) {
      uint32_t st = 0, ph = 0, ua = 0;  // ring slot and its phase bit
      for (int iu = 0;; ++iu, ++ua) {
        const int u = pair_unit(a, S, iu, pair, npairs, units, leader);
        if (!leader) pair_unit_release(a, S, iu);
        if (u < 0) break;
        int qp, r;
        unit_coords(a, u, &qp, &r);
        const int qt = 2 * qp + static_cast<int>(crank);
        tc::mbar_wait(&S.a_empty, (ua & 1u) ^ 1u);
        if (leader) expect_tx(&S.a_full, 2u * (static_cast<uint32_t>(a.KC) * kAChunkBytes + kAAugBytes));
        for (int kc = 0; kc < a.KC; ++kc) tma_2d_pair(a_s + kc * kAChunkBytes, &a.tmA, kc * 64, qt * kDenseM, a_full_l);
        tma_2d_pair(aa_s, &a.tmAa, 0, 0, a_full_l);
        int t0, t1;
        range_tiles(r, a.R, a.ntiles, &t0, &t1);
        for (int t = t0; t < t1; ++t) {
          const int row0 = static_cast<int>(a.off[a.tile_s0[t]]) + static_cast<int>(crank) * kHalfN;
          if (a.l2pf_ahead > 0 && t + a.l2pf_ahead < t1 && (t % a.l2pf_mod) == (pair % a.l2pf_mod)) {
            const int prow = static_cast<int>(a.off[a.tile_s0[t + a.l2pf_ahead]]) + static_cast<int>(crank) * kHalfN;
            for (int kc = 0; kc < a.KC; ++kc) tma_prefetch_l2(&a.tmB, kc * 64, prow);
            tma_prefetch_l2(&a.tmBa, 0, prow);
          }
          for (int kc = 0; kc <= a.KC; ++kc) {  // kc == KC: the norm chunk
            DPROF(0, tc::mbar_wait_sleep(&S.empty[st], ph ^ 1u));
            const uint32_t fb = full_l0 + st * 8u;
            if (a.debug == 4) {  // developer: no database loads (stale tiles; times the MMA issue alone)
              if (leader) tc::mbar_arrive(&S.full[st]);
            } else if (kc < a.KC) {
              if (leader) expect_tx(&S.full[st], 2u * kBChunkBytes);
              tma_2d_pair(ring_s + st * kBChunkBytes, &a.tmB, kc * 64, row0, fb);
            } else {
              if (leader) expect_tx(&S.full[st], 2u * kBAugBytes);
              tma_2d_pair(ring_s + st * kBChunkBytes, &a.tmBa, 0, row0, fb);
            }
            if (++st == static_cast<uint32_t>(NST)) {
              st = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // =========================== MMA issuer (one thread) ===========================
    // one thread runs the whole loop (no warp-wide waits or elections per MMA) with precomputed descriptors:
    // the start-address field is the low 14 bits of addr >> 4, so adding (byte offset >> 4) moves it while the
    // address stays below 256 KB
    if (lane == 0 && leader) {
      uint32_t st = 0, ph = 0, tile_ctr = 0, ua = 0;
      const uint32_t idesc = tc::idesc_f16_f32(2 * kDenseM, kDenseN);
      const uint64_t adesc0 = tc::sw128_desc(a_s), bdesc0 = tc::sw128_desc(ring_s);
      const uint64_t aadesc = sw32_desc(aa_s), badesc0 = sw32_desc(ring_s);
      const int KC = a.KC;
      for (int iu = 0;; ++iu, ++ua) {
        const int u = pair_unit(a, S, iu, pair, npairs, units, false);
        pair_unit_release(a, S, iu);
        if (u < 0) break;
        int qp, r;
        unit_coords(a, u, &qp, &r);
        tc::mbar_wait(&S.a_full, ua & 1u);
        tc::fence_after_sync();
        int t0, t1;
        range_tiles(r, a.R, a.ntiles, &t0, &t1);
        for (int t = t0; t < t1; ++t, ++tile_ctr) {
          const uint32_t acc = tile_ctr & 1u;
          DPROF(1, tc::mbar_wait(&S.tempty[acc], ((tile_ctr >> 1) & 1u) ^ 1u));
          tc::fence_after_sync();
          const uint32_t d_tmem = tmem + acc * kDenseN;
          for (int kc = 0; kc <= KC; ++kc) {
            DPROF(2, tc::mbar_wait(&S.full[st], ph));
            tc::fence_after_sync();
            const uint64_t soff = static_cast<uint64_t>((st * kBChunkBytes) >> 4);
            if (a.debug == 2) {
            } else if (kc < KC) {
              const uint64_t ad = adesc0 + static_cast<uint64_t>((kc * kAChunkBytes) >> 4), bd = bdesc0 + soff;
              umma_pair(d_tmem, ad, bd, idesc, kc ? 1u : 0u);
              umma_pair(d_tmem, ad + 2, bd + 2, idesc, 1u);
              umma_pair(d_tmem, ad + 4, bd + 4, idesc, 1u);
              umma_pair(d_tmem, ad + 6, bd + 6, idesc, 1u);
            } else {  // + alpha (h + l): the database row norms
              umma_pair(d_tmem, aadesc, badesc0 + soff, idesc, 1u);
            }
            umma_commit_pair(&S.empty[st]);
            if (++st == static_cast<uint32_t>(NST)) {
              st = 0;
              ph ^= 1u;
            }
          }
          umma_commit_pair(&S.tfull[acc]);
        }
        umma_commit_pair(&S.a_empty);  // the query tiles may be overwritten once these MMAs are done
      }
    }
    __syncwarp();
  } else if (warp == kInfoWarp) {
    // =========================== tile info (sets, columns, norms) ===========================
    uint32_t tile_ctr = 0;
    for (int iu = 0;; ++iu) {
      const int u = pair_unit(a, S, iu, pair, npairs, units, false);
      __syncwarp();
      if (lane == 0) pair_unit_release(a, S, iu);
      if (u < 0) break;
      int qp, r;
      unit_coords(a, u, &qp, &r);
      int t0, t1;
      range_tiles(r, a.R, a.ntiles, &t0, &t1);
      for (int t = t0; t < t1; ++t, ++tile_ctr) {
        const int slot = tile_ctr % kInfoSlotsD;
        DenseInfo& inf = S.info[slot];
        const int s0 = a.tile_s0[t], s1 = a.tile_s1[t];
        const int64_t row0 = a.off[s0];
        int16_t cl[(kDenseN + 31) / 32], ml[(kDenseN + 31) / 32];
#pragma unroll
        for (int c = 0; c < (kDenseN + 31) / 32; ++c) {
          const int j = lane + 32 * c;
          cl[c] = 0;
          ml[c] = 0;
          if (j < s1 - s0) {
            const int64_t v0 = a.off[s0 + j];
            cl[c] = static_cast<int16_t>(v0 - row0);
            ml[c] = static_cast<int16_t>(a.off[s0 + j + 1] - v0);
          }
        }
        tc::mbar_wait_sleep(&S.info_empty[slot], ((tile_ctr / kInfoSlotsD) & 1u) ^ 1u);
#pragma unroll
        for (int c = 0; c < (kDenseN + 31) / 32; ++c) {
          const int j = lane + 32 * c;
          if (j < kDenseN) {
            inf.col0[j] = cl[c];
            inf.mv[j] = ml[c];
          }
        }
        if (lane == 0) {
          inf.s0 = s0;
          inf.nsets = s1 - s0;
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.info_full[slot]);
      }
    }
  } else {
    // =========================== epilogue (warps 2 .. 2 + kEpiWarpsD - 1) ===========================
    const int quarter = warp & 3;
    const int sub = (warp - 2) >> 2;  // 0 .. kEpiSub-1: the quarter's warps take alternate sets
    const float INF = __int_as_float(0x7f800000);
    uint32_t tile_ctr = 0;
    unsigned long long n_surv = 0, n_emit = 0;  // statistics, flushed once (a per-survivor global atomic on one
                                                // address would serialise in L2)
    for (int iu = 0;; ++iu) {
      const int u = pair_unit(a, S, iu, pair, npairs, units, false);
      __syncwarp();
      if (lane == 0) pair_unit_release(a, S, iu);
      if (u < 0) break;
      int qp, r;
      unit_coords(a, u, &qp, &r);
      const int qt = 2 * qp + static_cast<int>(crank);
      const int prow = qt * kDenseM + quarter * 32 + lane;
      const int qid = a.lane_qid[prow];
      const bool valid = qid >= 0;
      const float qn = valid ? a.lane_qn[prow] : 0.0f;
      const unsigned segmask = __match_any_sync(0xffffffffu, qid);
      const float E = valid ? a.qE[qid] : 0.0f;
      const float* lq = valid ? a.lists + (static_cast<int64_t>(qid) * a.R + r) * kEpiSub * a.k : nullptr;
      float tau = valid ? vload_volatile(a.tau0 + qid) : INF;
      // dyn: inherit this warp's list of the previous range when that unit is complete.  The three warps of
      // a quarter see disjoint sets of the query, and an inherited list only ever continues in this range, so
      // the union of the current range's three lists holds distinct sets: its k-th is a valid tau over every
      // range run so far (the union never mixes ranges in dyn mode).
      if (a.dyn && r > 0) {
        int c;
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(c) : "l"(a.udone + static_cast<int64_t>(qp) * a.R + r - 1)
                     : "memory");
        if (c == 2 * kEpiWarpsD) {
          unsigned pend = __ballot_sync(0xffffffffu, valid);
          while (pend) {
            const int ld = __ffs(pend) - 1;
            pend &= ~__shfl_sync(0xffffffffu, segmask, ld);
            const int qq = __shfl_sync(0xffffffffu, qid, ld);
            float* dst = a.lists + ((static_cast<int64_t>(qq) * a.R + r) * kEpiSub + sub) * a.k;
            if (lane < a.k) dst[lane] = vload_volatile(dst - kEpiSub * a.k + lane);
          }
          __syncwarp();
        }
      }
      float other_k[kEpiSub - 1];  // the other warps' k-th bounds, loaded one tile ahead and used at the next
                                   // tile (the load latency stays hidden behind this tile's work)
#pragma unroll
      for (int o = 0; o < kEpiSub - 1; ++o) other_k[o] = INF;
      int t0, t1;
      range_tiles(r, a.R, a.ntiles, &t0, &t1);
      // candidate bitmap (top-T of the filter): this lane's query's bits of the tile's first two words, loaded
      // one tile ahead; a set outside them (a tile of many tiny sets) reads its word directly
      const uint32_t* mrow = (a.mask && valid) ? a.mask + static_cast<int64_t>(qid) * a.mask_stride : nullptr;
      auto mask_load = [&](int tt, uint64_t* bits, int* w0) {
        *bits = ~0ull;
        *w0 = 0;
        if (mrow && tt < t1) {
          *w0 = __ldg(a.tile_s0 + tt) >> 5;
          const uint32_t lo = __ldg(mrow + *w0);
          const uint32_t hi = *w0 + 1 <= a.mask_last_word ? __ldg(mrow + *w0 + 1) : 0u;
          *bits = static_cast<uint64_t>(lo) | (static_cast<uint64_t>(hi) << 32);
        }
      };
      uint64_t mbits_nx;
      int mw_nx;
      mask_load(t0, &mbits_nx, &mw_nx);
      for (int t = t0; t < t1; ++t, ++tile_ctr) {
        const uint32_t acc = tile_ctr & 1u;
        const int slot = tile_ctr % kInfoSlotsD;
        const uint64_t mbits = mbits_nx;
        const int mw0 = mw_nx;
        mask_load(t + 1, &mbits_nx, &mw_nx);
        // (developer BVSS_DENSE_DEBUG 8 .. 11 switch tau sources off: 8 none, 9 the own list, 10 + the other
        // warps' lists at insertion, 11 + the union)
        if (a.debug < 8) {
#pragma unroll
          for (int o = 0; o < kEpiSub - 1; ++o) tau = fminf(tau, other_k[o]);
        }
        // at the start of every unit and every 32 tiles (staggered): the k-th of
        if ((a.debug < 8 || a.debug == 11) &&
            (t == t0 || ((tile_ctr + a.refresh_stagger * static_cast<uint32_t>(sub)) & a.refresh_mask) == 0u)) {
          unsigned pend = __ballot_sync(0xffffffffu, valid);               // the union of the query's lists
          if (a.ukth_fast == 2 && a.dyn && kEpiSub * a.k <= 32) {
            // the loads of the first kPre query segments (their union values and running tau) are all issued
            // before any is used: one global round trip per refresh instead of two per segment
            constexpr int kPre = 4;
            float pv[kPre], pt[kPre];
            unsigned p = pend;
#pragma unroll
            for (int s2 = 0; s2 < kPre; ++s2) {
              pv[s2] = INF;
              pt[s2] = INF;
              if (p) {
                const int ld = __ffs(p) - 1;
                p &= ~__shfl_sync(0xffffffffu, segmask, ld);
                const int qq = __shfl_sync(0xffffffffu, qid, ld);
                pt[s2] = vload_volatile(a.tau0 + qq);
                if (lane < kEpiSub * a.k) pv[s2] = vload_volatile(a.lists + (static_cast<int64_t>(qq) * a.R + r) * kEpiSub * a.k + lane);
              }
            }
#pragma unroll
            for (int s2 = 0; s2 < kPre; ++s2) {
              if (pend) {
                const int ld = __ffs(pend) - 1;
                const unsigned sm = __shfl_sync(0xffffffffu, segmask, ld);
                pend &= ~sm;
                const int qq = __shfl_sync(0xffffffffu, qid, ld);
                const float uk = ukth_rank(pv[s2], a.k, lane);
                const float tr = pt[s2];
                if ((sm >> lane) & 1u) tau = fminf(tau, fminf(uk, tr));
                if (lane == ld && tau < tr) atomicMin(reinterpret_cast<int*>(a.tau0) + qq, __float_as_int(tau));
              }
            }
          }
          while (pend) {
            const int ld = __ffs(pend) - 1;
            const unsigned sm = __shfl_sync(0xffffffffu, segmask, ld);
            pend &= ~sm;
            const int qq = __shfl_sync(0xffffffffu, qid, ld);
            const int nr = a.dyn ? 1 : (a.R < 8 ? a.R : 8);
            const float tr = vload_volatile(a.tau0 + qq);  // (issued before the list loads: both in flight at once)
            const float uk = union_kth(a.lists + static_cast<int64_t>(qq) * a.R * kEpiSub * a.k, a.R, r, nr, a.k, lane,
                                       a.dyn ? -1 : 1, a.ukth_fast != 0);
            if ((sm >> lane) & 1u) tau = fminf(tau, fminf(uk, tr));
            if (lane == ld && tau < tr) atomicMin(reinterpret_cast<int*>(a.tau0) + qq, __float_as_int(tau));
          }
        }
        if (valid) {
#pragma unroll
          for (int o = 1; o < kEpiSub; ++o) other_k[o - 1] = vload_volatile(lq + ((sub + o) % kEpiSub) * a.k + a.k - 1);
        }
        float thr = tau + E;
        DPROF(3, tc::mbar_wait_sleep(&S.info_full[slot], (tile_ctr / kInfoSlotsD) & 1u));
        const DenseInfo& inf = S.info[slot];
        DPROF(4, tc::mbar_wait_sleep(&S.tfull[acc], (tile_ctr >> 1) & 1u));
        tc::fence_after_sync();
        const int s0 = inf.s0, nsets = inf.nsets;
        const uint32_t tb = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + acc * kDenseN;
        // one set of the tile for this warp's lane quarter (its columns read into `cols`; a software-pipelined
        // form that issued the next set's reads before this set's math needed a second column buffer and
        // spilled ~1 KB per thread at the 128-register cap, so the reads stay synchronous)
        auto do_set = [&](int js, Cols& cols) {
          const int i = s0 + js;
          const int col0 = inf.col0[js];
          const int mv = inf.mv[js];
          float m = -INF;  // max_v acc (kappa < 0: the min over v of D^2)
          for (int j0 = 0; j0 < mv; j0 += CH) {
            const int mvc = min(CH, mv - j0);
            load_set(tb + static_cast<uint32_t>(col0 + j0), mvc, cols);
            m = fmaxf(m, set_max(cols, mvc));
          }
          const float rq = fmaxf(fmaf(a.kappa, m, qn), 0.0f);
          bool cand = true;  // set i is in this lane's query's candidate bitmap (always without a bitmap)
          if (mrow) {
            const int bi = i - 32 * mw0;
            cand = bi < 64 ? ((mbits >> bi) & 1ull) != 0ull : ((__ldg(mrow + (i >> 5)) >> (i & 31)) & 1u) != 0u;
          }
          const unsigned pass = __ballot_sync(0xffffffffu, !valid || (rq <= thr && cand));
          unsigned sb = __ballot_sync(0xffffffffu, valid && (pass & segmask) == segmask);
          if (a.debug == 3) sb = 0u;  // developer: no survivor work (times the base epilogue)
          while (sb) {  // warp-uniform: one surviving query segment at a time
            const int leader = __ffs(sb) - 1;
            const unsigned smask = __shfl_sync(0xffffffffu, segmask, leader);
            sb &= ~smask;
            const int q = __shfl_sync(0xffffffffu, qid, leader);
            const bool inseg = (smask >> lane) & 1u;
            const float A = __uint_as_float(__reduce_max_sync(0xffffffffu, inseg ? __float_as_uint(rq) : 0u));
            const float Eq = __shfl_sync(0xffffffffu, E, leader);
            const float tq = __shfl_sync(0xffffffffu, tau, leader);
            // B is only needed while h = max(A, B) <= tq + Eq: above it the set is neither inserted (ub > tq)
            // nor emitted (h - Eq > tq >= the tau after any insertion), so the column scan may stop early
            const float lim = tq + Eq;
            float B;
            if (mv <= CH) {
              B = set_colmin_max(cols, mv, a.kappa, qn, inseg, lim);
            } else {
              B = 0.0f;
              for (int j0 = 0; j0 < mv && B <= lim; j0 += CH) {
                Cols cb;
                const int mvc = min(CH, mv - j0);
                load_set(tb + static_cast<uint32_t>(col0 + j0), mvc, cb);
                B = fmaxf(B, set_colmin_max(cb, mvc, a.kappa, qn, inseg));
              }
            }
            const float h = fmaxf(A, B);
            const float ub = h + Eq;
            float newtau = tq;
            ++n_surv;
            if (ub < tq) {  // warp-uniform: insert ub into this warp's sorted list of k bounds, lane-parallel
              const float* lqq = a.lists + (static_cast<int64_t>(q) * a.R + r) * kEpiSub * a.k;
              float* ownq = const_cast<float*>(lqq) + sub * a.k;
              const float old = lane < a.k ? ownq[lane] : INF;
              const float oth = lane < kEpiSub - 1 && a.debug != 9 ? vload_volatile(lqq + ((sub + 1 + lane) % kEpiSub) * a.k + a.k - 1)
                                                   : INF;
              const int pos = __popc(__ballot_sync(0xffffffffu, lane < a.k && old <= ub));
              const float up = __shfl_up_sync(0xffffffffu, old, 1);
              const float nw = lane < pos ? old : (lane == pos ? ub : up);
              if (lane < a.k) ownq[lane] = nw;
              const float kth = __shfl_sync(0xffffffffu, nw, a.k - 1);
              // (min with tq: the warp's tau may be tighter than its lists, e.g. from the union)
              newtau = fminf(tq, fminf(kth, __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(oth)))));
            }
            if (lane == leader && h - Eq <= newtau) {
              const int slot = atomicAdd(a.cnt + q, 1);
              if (slot < a.cap) {
                a.ids[static_cast<int64_t>(q) * a.cap + slot] = static_cast<int32_t>(a.id_base + i);
                a.vals[static_cast<int64_t>(q) * a.cap + slot] = h;
              }
              ++n_emit;
            }
            if (inseg && a.debug != 8) {
              tau = newtau;
              thr = tau + E;
            }
          }
        };
        const int js0 = (a.debug == 1 || a.debug == 4) ? nsets : sub;
        // the quarter's warps take the tile's sets in turn (static: a shared-memory work counter per set cost
        // more than the imbalance it removed, 2795 vs 2730 ms per bench step, profiles/r02/s3/ab_static_split.log)
        for (int js = js0; js < nsets; js += kEpiSub) {
          Cols cols;  // (sets of <= CH rows keep their columns in registers for the survivor's B)
          do_set(js, cols);
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) {
          if (leader) tc::mbar_arrive(&S.tempty[acc]);  // the leader's barrier (its MMA thread reuses the accumulator)
          else arrive_remote(tempty_l0 + acc * 8u);
          tc::mbar_arrive(&S.info_empty[slot]);
        }
      }
      // the unit's final tau of each query segment -> the query's running tau
      if (valid && lane == __ffs(segmask) - 1 && a.debug < 8)
        atomicMin(reinterpret_cast<int*>(a.tau0) + qid, __float_as_int(tau));
      if (a.dyn) {  // this warp's lists of the unit are final (release: the next range may inherit them)
        __threadfence();
        __syncwarp();
        if (lane == 0)
          asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.udone + static_cast<int64_t>(qp) * a.R + r)
                       : "memory");
      }
    }
    unsigned int ne = static_cast<unsigned int>(n_emit);
    ne = __reduce_add_sync(0xffffffffu, ne);  // emissions were counted by the segment leaders
    if (a.stat && lane == 0) {
      atomicAdd(a.stat, n_surv);
      atomicAdd(a.stat + 1, static_cast<unsigned long long>(ne));
    }
  }
  if (a.prof && lane == 0) atomicAdd(&a.prof[8 + (warp == 0 ? 0 : warp == 1 ? 1 : warp == kInfoWarp ? 2 : 3)],
                                     (unsigned long long)(clock64() - t_start));
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync_all();  // neither CTA leaves while the other still signals its barriers or uses the pair's TMEM
  if (warp == 1) {
    tc::fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ------------------------------------------------------------ helper kernels --
// fp16 copy of the database, x / S (S a power of two >= max|x|), zero-padded to dpad columns
__global__ void dense_db_operand_kernel(const float* __restrict__ V, int64_t nvec, int d, int dpad, float inv_s,
                                        __half* __restrict__ hd) {
  const int64_t total = nvec * dpad;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = e / dpad;
    const int c = static_cast<int>(e - v * dpad);
    hd[e] = __float2half_rn(c < d ? V[v * d + c] * inv_s : 0.0f);
  }
}

// the norm chunk of the database operand: va[v] = (h, l, 0 x 14), h + l = the fp16 split of |v|^2 / S_db^2
__global__ void dense_norm_operand_kernel(const float* __restrict__ vn, int64_t nvec, float inv_s2,
                                          __half* __restrict__ va) {
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < nvec;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float x = vn[v] * inv_s2;
    const __half h = __float2half_rn(x);
    const __half l = __float2half_rn(x - __half2float(h));
    __half2* row = reinterpret_cast<__half2*>(va + v * 16);
    row[0] = __halves2half2(h, l);
#pragma unroll
    for (int i = 1; i < 8; ++i) row[i] = __float2half2_rn(0.0f);
  }
}

// packed query rows: qd[row] = fp16(q / S_q) (zero rows for padding), lane meta
__global__ void dense_query_operand_kernel(const float* __restrict__ Qv, const float* __restrict__ qnorm,
                                           const int32_t* __restrict__ rowmap /*[rows]: query vector or -1*/,
                                           const int32_t* __restrict__ rowq /*[rows]: query or -1*/, int64_t rows,
                                           int d, int dpad, float inv_s, __half* __restrict__ qd,
                                           int32_t* __restrict__ lane_qid, float* __restrict__ lane_qn) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; r < rows;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int32_t v = rowmap[r];
    for (int c = lane; c < dpad; c += 32)
      qd[r * dpad + c] = __float2half_rn((v >= 0 && c < d) ? Qv[static_cast<int64_t>(v) * d + c] * inv_s : 0.0f);
    if (lane == 0) {
      lane_qid[r] = v >= 0 ? rowq[r] : -1;
      lane_qn[r] = v >= 0 ? qnorm[v] : 0.0f;
    }
  }
}

// per-query error bound E = c1 Mq Mv + c2 (Mq^2 + Mv^2), Mq^2 = max squared norm of the query's vectors
__global__ void dense_query_bound_kernel(const int64_t* __restrict__ qoff, const float* __restrict__ qnorm, int nq,
                                         float c1, float c2, float vmax2, float* __restrict__ qE) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  float m2 = 0.0f;
  for (int64_t v = qoff[q]; v < qoff[q + 1]; ++v) m2 = fmaxf(m2, qnorm[v]);
  qE[q] = c1 * sqrtf(m2) * sqrtf(vmax2) + c2 * (m2 + vmax2);
}

__global__ void dense_fill_kernel(float* __restrict__ x, int64_t n, float v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] = v;
}

// sets the tiles cannot hold (> 256 rows): appended to every query's list with the K6 exact sentinel
// (every one is recomputed exactly), honouring the candidate bitmap
__global__ void dense_append_huge_kernel(const int32_t* __restrict__ huge, int nhuge, const uint32_t* __restrict__ mask,
                                         int64_t mask_stride, int nq, int64_t id_base, int32_t* __restrict__ cnt,
                                         int32_t* __restrict__ ids, float* __restrict__ vals, int cap) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  int c = 0;
  for (int h = 0; h < nhuge; ++h) {
    const int i = huge[h];
    if (mask && ((mask[static_cast<int64_t>(q) * mask_stride + (i >> 5)] >> (i & 31)) & 1u) == 0u) continue;
    if (c < cap) {
      ids[static_cast<int64_t>(q) * cap + c] = static_cast<int32_t>(id_base + i);
      vals[static_cast<int64_t>(q) * cap + c] = -1.0f;  // refine.cu kExactSentinel
    }
    ++c;
  }
  cnt[q] = c;
}

// ------------------------------------------------------------------ host --
static int encode_map(CUtensorMap* map, const void* base, int64_t rows, int dpad, int box_rows, int box_cols = 64,
                      CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    BVSS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) BVSS_FAIL(BVSS_ECUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(dpad), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(dpad) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) BVSS_FAIL(BVSS_ECUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return BVSS_OK;
}

int dense_max_dpad() { return 512; }
int dense_tile_rows() { return kDenseN; }
int dense_epi_sub() { return kEpiSub; }

// stages that fit next to a query tile of KC chunks
static int dense_stages(int KC, size_t* smem) {
  const size_t budget = 227 * 1024 - sizeof(DenseCtl) - 1024;  // static shared memory (DenseCtl, 1 KB aligned)
  const size_t fixed = 1024 + static_cast<size_t>(KC) * kAChunkBytes + kAAugBytes;
  if (fixed + 2 * kBChunkBytes > budget) return 0;
  int st = static_cast<int>((budget - fixed) / kBChunkBytes);
  if (st > kDenseMaxStages) st = kDenseMaxStages;
  *smem = fixed + static_cast<size_t>(st) * kBChunkBytes;
  return st;
}

int launch_dense_db_operand(const float* V, int64_t nvec, int d, int dpad, float inv_s, __half* hd, int num_sms,
                            cudaStream_t st) {
  if (nvec <= 0) return BVSS_OK;
  dense_db_operand_kernel<<<num_sms * 16, 256, 0, st>>>(V, nvec, d, dpad, inv_s, hd);
  return post_launch("dense_db_operand_kernel", st);
}

int launch_dense_norm_operand(const float* vn, int64_t nvec, float inv_s2, __half* va, int num_sms, cudaStream_t st) {
  if (nvec <= 0) return BVSS_OK;
  dense_norm_operand_kernel<<<num_sms * 8, 256, 0, st>>>(vn, nvec, inv_s2, va);
  return post_launch("dense_norm_operand_kernel", st);
}

int launch_dense_query_operand(const float* Qv, const float* qnorm, const int32_t* rowmap, const int32_t* rowq,
                               int64_t rows, int d, int dpad, float inv_s, __half* qd, int32_t* lane_qid,
                               float* lane_qn, int num_sms, cudaStream_t st) {
  if (rows <= 0) return BVSS_OK;
  dense_query_operand_kernel<<<num_sms * 4, 256, 0, st>>>(Qv, qnorm, rowmap, rowq, rows, d, dpad, inv_s, qd, lane_qid,
                                                          lane_qn);
  return post_launch("dense_query_operand_kernel", st);
}

int launch_dense_prep(const int64_t* qoff, const float* qnorm, int nq, float c1, float c2, float vmax2, float* qE,
                      float* lists, int64_t nlist, int32_t* cnt, const int32_t* huge, int nhuge, const uint32_t* mask,
                      int64_t mask_stride, int64_t id_base, int32_t* ids, float* vals, int cap, int num_sms,
                      cudaStream_t st) {
  dense_query_bound_kernel<<<ceil_div(nq, 128), 128, 0, st>>>(qoff, qnorm, nq, c1, c2, vmax2, qE);
  BVSS_TRY(post_launch("dense_query_bound_kernel", st));
  dense_fill_kernel<<<num_sms * 4, 256, 0, st>>>(lists, nlist, INFINITY);
  BVSS_TRY(post_launch("dense_fill_kernel", st));
  dense_append_huge_kernel<<<ceil_div(nq, 128), 128, 0, st>>>(huge, nhuge, mask, mask_stride, nq, id_base, cnt, ids,
                                                              vals, cap);
  return post_launch("dense_append_huge_kernel", st);
}

int launch_dense_hausdorff(const __half* qd, int ntq, const __half* hd, int64_t nvec, int dpad, int ntiles,
                           const int32_t* tile_s0, const int32_t* tile_s1, const int64_t* off, const __half* va,
                           const __half* qa,
                           const int32_t* lane_qid, const float* lane_qn, const float* qE, float* tau0,
                           float kappa, float alpha, int k, int R, float* lists, int32_t* cnt, int32_t* ids,
                           float* vals, int cap,
                           const uint32_t* mask, int64_t mask_stride, int64_t id_base, unsigned long long* stat,
                           int dyn, int* unit_ctr, int* udone, int num_sms, cudaStream_t st) {
  if (ntq <= 0 || ntiles <= 0) return BVSS_OK;
  if (dpad % 64 || dpad > dense_max_dpad()) BVSS_FAIL(BVSS_EUNSUPPORTED, "dense path needs dpad <= 512");
  DenseArgs a;
  std::memset(&a, 0, sizeof(a));
  BVSS_TRY(encode_map(&a.tmA, qd, static_cast<int64_t>(ntq) * kDenseM, dpad, kDenseM));
  BVSS_TRY(encode_map(&a.tmB, hd, nvec, dpad, kHalfN));
  BVSS_TRY(encode_map(&a.tmAa, qa, kDenseM, 16, kDenseM, 16, CU_TENSOR_MAP_SWIZZLE_32B));
  BVSS_TRY(encode_map(&a.tmBa, va, nvec, 16, kHalfN, 16, CU_TENSOR_MAP_SWIZZLE_32B));
  a.KC = dpad / 64;
  size_t smem = 0;
  a.stages = dense_stages(a.KC, &smem);
  if (a.stages < 2) BVSS_FAIL(BVSS_EUNSUPPORTED, "dense path: no room for two stages");
  a.ntq = ntq;
  a.R = R;
  a.ntiles = ntiles;
  a.tile_s0 = tile_s0;
  a.tile_s1 = tile_s1;
  a.off = off;
  a.lane_qid = lane_qid;
  a.lane_qn = lane_qn;
  a.qE = qE;
  a.tau0 = tau0;
  a.kappa = kappa;
  (void)alpha;  // (the query tile's norm chunk comes from qa by TMA)
  a.k = k;
  a.lists = lists;
  a.cnt = cnt;
  a.ids = ids;
  a.vals = vals;
  a.cap = cap;
  a.mask = mask;
  a.mask_stride = mask_stride;
  if (mask) {  // (tile_s1 is a device array: the last set of the last tile comes back once per launch)
    int last = 0;
    BVSS_CUDA(cudaMemcpyAsync(&last, tile_s1 + ntiles - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    BVSS_CUDA(cudaStreamSynchronize(st));
    a.mask_last_word = (last - 1) >> 5;
  }
  a.id_base = id_base;
  a.stat = stat;
  a.dyn = dyn;
  a.unit_ctr = unit_ctr;
  a.udone = udone;
  if (dyn) {
    BVSS_CUDA(cudaMemsetAsync(unit_ctr, 0, sizeof(int), st));
    BVSS_CUDA(cudaMemsetAsync(udone, 0, static_cast<size_t>(ntq / 2) * R * sizeof(int), st));
  }
  {
    const char* e = getenv("BVSS_DENSE_DEBUG");
    a.debug = e ? atoi(e) : 0;
    int per = 32, stag = 8;
    if (const char* f = getenv("BVSS_DENSE_REFRESH")) sscanf(f, "%d,%d", &per, &stag);
    if (per < 1 || (per & (per - 1))) BVSS_FAIL(BVSS_EINVAL, "BVSS_DENSE_REFRESH: the period must be a power of two");
    a.refresh_mask = static_cast<uint32_t>(per - 1);
    a.refresh_stagger = static_cast<uint32_t>(stag);
    const char* g = getenv("BVSS_DENSE_UKTH");
    a.ukth_fast = g ? atoi(g) : 2;
    a.l2pf_ahead = 0;
    a.l2pf_mod = 1;
    if (const char* f = getenv("BVSS_DENSE_L2PF")) sscanf(f, "%d,%d", &a.l2pf_ahead, &a.l2pf_mod);
    if (a.l2pf_mod < 1) a.l2pf_mod = 1;
  }
  static unsigned long long* prof = nullptr;
  a.prof = nullptr;
  if (getenv("BVSS_DENSE_PROF")) {
    if (!prof) cudaMalloc(&prof, 16 * sizeof(unsigned long long));
    cudaMemsetAsync(prof, 0, 16 * sizeof(unsigned long long), st);
    a.prof = prof;
  }
  if (ntq % 2) BVSS_FAIL(BVSS_EINVAL, "dense kernel: the query tiles come in pairs (ntq must be even)");
  const int units = (ntq / 2) * R;
  int pairs = num_sms / 2;
  if (pairs > units) pairs = units;
  auto kern = dense_hausdorff_kernel;
  BVSS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
  cfg.blockDim = dim3(kDenseThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BVSS_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  BVSS_TRY(post_launch("dense_hausdorff_kernel", st));
  if (a.prof) {  // developer instrumentation: per-CTA Mcycles per role and wait (epilogue: per warp)
    unsigned long long h[16];
    cudaMemcpyAsync(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const double g = 2.0 * pairs, ew = g * kEpiWarpsD;
    fprintf(stderr,
            "[dense prof] Mcycles per CTA: producer %.1f (empty wait %.1f) | mma %.1f (tempty %.1f, full %.1f) | "
            "info %.1f | per epilogue warp %.1f (info wait %.1f, tfull wait %.1f)\n",
            h[8] / g / 1e6, h[0] / g / 1e6, h[9] / (g / 2) / 1e6, h[1] / (g / 2) / 1e6, h[2] / (g / 2) / 1e6,
            h[10] / g / 1e6, h[11] / ew / 1e6, h[3] / ew / 1e6, h[4] / ew / 1e6);
  }
  return BVSS_OK;
}

}  // namespace bvss
