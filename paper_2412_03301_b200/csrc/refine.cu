// refine.cu — K5: Hausdorff refinement of the T candidates of every query on the
// 5th-generation tensor cores (Alg 6 lines 19-22; Def 4).
//
// For a query Q (m_q vectors) and a run of its candidate sets, the Gram matrix
// G = Q V^T is formed by tcgen05.mma with the QUERY as the A operand (M = 128:
// the query rows replicated 128/(32*ceil(m_q/32)) times, one replica per TMEM
// lane quarter) and 256 packed candidate rows as the B operand (N = 256), K = d.
// Measured on B200 (tools/microbench_umma.cu, 148 CTAs) a tcgen05.mma M=128 K=16
// costs ~200-220 cycles whatever N is (64..256; A in shared memory or in TMEM), so
// N = 256 candidate rows per instruction is what keeps the tensor pipe off the
// critical path.  Operands are the scaled fp16 split made at
// build time, x = s (hi + lo) + r with s a power of two >= max|x|; terms = 1
// issues hi*hi (|error| <= ~2^-10 |x||y|), terms = 3 hi*hi + hi*lo + lo*hi.
//
// Epilogue: TMEM lane = query row, column = candidate row.  One warp per
// candidate set (sets are whole inside a tile): per lane the min over the set's
// columns of D^2 = |q|^2 + |v|^2 - 2 s_q s_v g (clamped at 0), per column the
// min over lanes (redux.sync), then
//     H^2 = max( max_q min_v D^2 , max_v min_q D^2 )
// with full-mask redux.sync max/min; no shared-memory round trip when m_q <= 32.
// K6 recomputes the final top-k window exactly in fp32 (topk.cu).
//
// Gather.  The fp16 copies are stored super-chunk-major and
// pre-swizzled: [KS][P/8][KCS][8 rows][64 halves] (KCS consecutive 128-byte
// K-chunks of each 8-row group together, 16-byte units of row p permuted
// u -> u ^ (p & 7)).  Every set starts on an 8-aligned padded row, so the
// (set, super-chunk) slab is ONE contiguous run of ceil8(m) x KCS x 128 bytes
// and lands, by a single cp.async.bulk, as ready-made SWIZZLE_128B K-major atoms
// with SBO = KCS x 1 KB.  (Measured: lane-parallel random bulk copies of >= 5 KB
// reach ~7 TB/s on B200, 2.5 KB copies only ~4 TB/s.)  Queries use the same
// layout with 8-aligned rows.
//
// CTA = 13 warps: warp 6 builds the item tables (work items, set sizes, tile
// packing), warp 7 the tile infos (|v|^2 and scale of every column), warps 0
// and 12 issue the bulk copies of a stage (even / odd entries; one cp.async.bulk
// issues per active lane), warp 1 owns TMEM and issues the MMAs (one thread),
// warps 2-5 and 8-11 run the epilogue (two per TMEM lane quarter).
// Accumulators (128 lanes x 256 columns) are double-buffered in TMEM (512
// columns); item tables, tile infos and stages are handed over with mbarriers,
// so the persistent loop has no CTA-wide barrier.  The kernel is a template on
// the rerank metric (Hausdorff / MeanMin / Min) and on the developer switches
// (EXPER), which stay out of the default instantiation's hot loops.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "tc.cuh"

namespace bvss {

constexpr int kTileRows = 256;   // candidate rows per tile (MMA N)
constexpr int kItemCands = 128;  // candidates per work item
constexpr int kKChunk = 64;      // fp16 per K-chunk = 128 bytes = one SW128 row
constexpr int kEpiWarps = 8;           // warps 2-5 and 8-11 (two per TMEM lane quarter)
constexpr int kProducers = 2;  // copy-producer warps: 0, 12 (measured: 3 is no faster)
constexpr int kRefineThreads = 32 * (11 + kProducers);  // 0 copy, 1 MMA, 2-5 epilogue, 6 table, 7 tile info, 8-11 epilogue,
                                          // 12 second copy producer (the copies of a stage are split in two)
constexpr int kMaxQ = 128;       // query rows the tensor path handles (M); larger query sets take the exact path
// tensor-core value of a candidate the tensor path does not take (a database set > 256 rows, a query set >
// 128 rows): negative, so that K6 (topk.cu) keeps it out of the k-th-smallest select (as uint32 bits it orders
// after every finite non-negative value) and always inside the exact window (-1 <= W)
constexpr float kExactSentinel = -1.0f;
constexpr int kMaxStages = 8;
constexpr int kInfoSlots = 4;
constexpr int kMaxSetsPerTile = kTileRows / 8;

struct RefineArgs {
  const __half* hs;      // [KS][prows/8][KCS][8][64] super-chunk-major, pre-swizzled, 8-row-aligned sets
  const __half* ls;
  const float* vscale;   // [prows] power-of-two scale of each padded row
  int64_t pgroups;       // prows / 8
  const int64_t* pbase;  // [n] first padded row of each set
  const float* vnorm;    // [nvec] squared norms (unpadded index)
  const int64_t* off;    // [n+1]
  int KC, KCS;
  const __half* qhs;     // [KS][qrows/8][KCS][8][64], 8-aligned queries
  const __half* qls;
  const float* qscale;   // [qrows]
  int64_t qgroups;
  const int64_t* qrow;   // [nq] first padded row of each query
  const float* qnorm;
  const int64_t* qoff;
  const int32_t* cand;   // [nq][T] global ids (-1 padded)
  const int32_t* count;  // [nq] valid candidates per query (may be null: T)
  int T;
  int nq;
  int64_t id_base;
  float* out_h2;  // [nq][T]; 0 for sets the tensor path does not take (> 256 rows): forces the exact fix-up
  int terms;
  int stages;
  uint32_t stage_bytes;
  uint32_t a_bytes;  // one A piece of a stage: 128 rows x KCS x 128 B
  uint32_t b_bytes;  // one B piece of a stage: 256 rows x KCS x 128 B
  int items_per_query;
  int total_items;
  int* work_counter;
  unsigned long long* rows_counter;  // candidate rows gathered (stats)
  unsigned long long* prof;          // developer per-role cycle counters (env BVSS_REFINE_PROF) or null
  // TMA maps over the pre-swizzled operand viewed as [KS][P/8][KCS][8 rows][64 halves] with box
  // (64 halves x h rows) of one K-chunk of one 8-row group, h = 1..8: the last, partial group of a set
  // is fetched without its padding rows
  CUtensorMap tm_hi[8], tm_lo[8];
  int tma;                           // developer switch BVSS_REFINE_TMA=1: partial groups by TMA (measured slower)
  int tail;                          // read only the m real rows of every set (no 8-row padding): BVSS_REFINE_TAIL
  // group mode (all m_q <= 32): an item is (query block, database range, group of 4 queries); the 4
  // queries take one TMEM lane quarter each and share the B tiles of their candidates in the range, and
  // items run range-major inside a query block so the CTAs in flight gather the same range (L2 reuse)
  int group;
  int qblock;                        // queries per block (multiple of 4)
  int64_t range_sets;                // database sets per range
  int nranges;
  int64_t n_local;                   // sets of this shard
  const int32_t* bounds;             // [nq][nranges+1] first candidate position of each range (range_bounds_kernel)
  const float2* qpack;               // [nq][32] (|q_i|^2, 2 scale_i) per query row, 0 past m_q (group mode)
  const longlong2* qmeta;            // [nq] (m_q, first padded query row) (group mode)
  int prefetch;                      // developer switch: L2 prefetch of the next tile's rows (env BVSS_REFINE_PREFETCH=1)
  // A in TMEM (terms = 1, query-major, dpad <= 512): the query is copied once per work item into TMEM
  // columns [acol, acol + dpad/2) by tcgen05.cp, replicated over the lane quarters by the copy itself
  // (32x128b.warpx4 / 64x128b.warpx2::02_13 / 128x128b); the stage ring then carries B only, and the
  // two accumulators take N = ncols columns each (ncols = 160 at dpad = 384)
  int atmem;
  int metric;                        // 0 Hausdorff (H^2), 1 MeanMin (mean_q sqrt(min_v D^2)), 2 Min (min D^2)
  float* out_err;                    // MeanMin: [nq][T] bound on |approx - exact| per candidate (topk.cu window)
  float c1, c2, vmax2;               // the squared-distance error bound E = c1 |q||v| + c2 (|q|^2 + |v|^2)
  int ncols;                         // candidate rows per tile (MMA N); 256 when A is in shared memory
  uint32_t acol;                     // first TMEM column of the resident query (atmem)
};

struct ItemTable {
  int nc;  // candidates in the item; -1 = no more work
  int q, c0, mq, rep_rows, reps, ntiles;
  int64_t q0, qrow;
  int gq0, gqend;     // group mode: the item's queries [gq0, gqend); tile t holds queries gq0 + 4 tile_grp[t] + quarter
  int gmq[32];        // group mode: m_q and first padded row of the item's 32 queries (0 / unused past gqend)
  int64_t gqr[32];
  int8_t tile_grp[kItemCands + 1];
  int8_t ent_quarter[kItemCands];  // group mode: lane quarter (query) of each entry
  int32_t tile_first[kItemCands + 1];  // first table entry of each tile (entries are in tile order)
  int32_t ent_cand[kItemCands];        // candidate index (within the item) of each entry
  int16_t ent_col[kItemCands];         // column (B row) where the set starts in its tile
  int16_t ent_m[kItemCands];           // vectors in the set
  int64_t ent_vbase[kItemCands];       // first (unpadded) vector index
  int64_t ent_pbase[kItemCands];       // first padded row
  float qn[kMaxQ];                     // |q_i|^2
  float qs2[kMaxQ];                    // 2 * scale of query row i
  float E;                             // squared-distance error bound of the item's query (MeanMin)
};

struct TileInfo {
  int first, count, pad0, pad1;  // entries of the item table in this tile (pad: 16-byte aligned vn/vs)
  float vn[kTileRows];       // |v|^2 of each column (candidate row)
  float vs[kTileRows];       // scale of each column
};

struct RefineCtl {
  ItemTable tab[2];
  TileInfo info[kInfoSlots];
  uint32_t hq[kEpiWarps][kMaxSetsPerTile];  // general path (m_q > 32): cross-warp partials
  uint32_t cm[kEpiWarps][kTileRows];
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint64_t tab_full[2];
  uint64_t tab_empty[2];
  uint64_t info_full[kInfoSlots];
  uint64_t info_empty[kInfoSlots];
  uint32_t tmem_base;
};

#define PROF_WAIT(slot, call)                                                        \
  do {                                                                               \
    if (a.prof) {                                                                    \
      const long long t0_ = clock64();                                               \
      call;                                                                          \
      if (lane == 0) atomicAdd(&a.prof[slot], (unsigned long long)(clock64() - t0_)); \
    } else {                                                                         \
      call;                                                                          \
    }                                                                                \
  } while (0)

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// one box of a 5D tensor map into shared memory, completion on an mbarrier (transaction bytes)
__device__ __forceinline__ void tma_5d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                       uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// SW128 K-major descriptor with a given stride between 8-row groups (SBO, bytes)
__device__ __forceinline__ uint64_t sw128_desc_sbo(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}
__device__ __forceinline__ void tmem_ld16f(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  tc::tmem_ld16(taddr, r);
  tc::tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// METRIC: 0 Hausdorff, 1 MeanMin, 2 Min; EXPER: the developer switches (A in TMEM, padding-free tails, TMA
// tails, range-major group items, L2 prefetch, narrower tiles) -- compiled out of the default instantiation,
// whose hot loops they measurably slow down (tools/ab_lib.sh)
template <int METRIC, bool EXPER>
__global__ void __launch_bounds__(kRefineThreads, 1) refine_tc_kernel(const __grid_constant__ RefineArgs a) {
  const bool x_atmem = EXPER && a.atmem, x_tail = EXPER && a.tail, x_tma = EXPER && a.tma, x_group = EXPER && a.group,
             x_prefetch = EXPER && a.prefetch;
  const int x_ncols = EXPER ? a.ncols : kTileRows;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ RefineCtl S;
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t ring_s = smem_u32(ring);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NST = a.stages;

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&S.full[s], 1);
      tc::mbar_init(&S.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&S.tfull[b], 1);
      tc::mbar_init(&S.tempty[b], kEpiWarps);
      tc::mbar_init(&S.tab_full[b], 1);
      tc::mbar_init(&S.tab_empty[b], kProducers + 3);  // copy producers + MMA warp + epilogue + tile-info warp
    }
    for (int s = 0; s < kInfoSlots; ++s) {
      tc::mbar_init(&S.info_full[s], 1);
      tc::mbar_init(&S.info_empty[s], kEpiWarps);
    }
    tc::fence_mbar_init();
  }
  for (int i = tid; i < kEpiWarps * kTileRows; i += blockDim.x) (&S.cm[0][0])[i] = METRIC == 1 ? 0u : 0x7f800000u;
  for (int i = tid; i < kEpiWarps * kMaxSetsPerTile; i += blockDim.x) (&S.hq[0][0])[i] = 0u;
  if (warp == 1) tc::tmem_alloc(&S.tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = S.tmem_base;
  const int KCS = a.KCS, KS = a.KC / a.KCS;
  const bool three = EXPER && a.terms == 3;  // the 3-term Gram runs in the EXPER instantiation
  const uint32_t sbo = static_cast<uint32_t>(KCS) * 1024u;
  const long long t_role0 = clock64();

  if (warp == 6 && x_group) {
    // ====== item tables, group mode: (query block, range, 32 queries); tiles hold 4 queries (one per lane quarter) ======
    int q0 = 0, qend = 0;
    int pl = 0, cntq = 0, incl = 0;  // this lane's query: first position of its slice, slice length, inclusive prefix
    int cursor = 0, total = 0;
    const int GI = (a.qblock + 31) / 32;  // 32-query chunks per block
    for (uint32_t it = 0;; ++it) {
      const int tb = it & 1;
      ItemTable& t = S.tab[tb];
      PROF_WAIT(0, tc::mbar_wait(&S.tab_empty[tb], ((it >> 1) & 1u) ^ 1u));
      bool done = false;
      while (cursor >= total) {  // next item with at least one candidate
        int item = 0;
        if (lane == 0) item = atomicAdd(a.work_counter, 1);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= a.total_items) {
          done = true;
          break;
        }
        const int gi = item % GI;
        const int br = item / GI;
        const int r = br % a.nranges, b = br / a.nranges;
        q0 = b * a.qblock + 32 * gi;
        qend = min(min(a.nq, (b + 1) * a.qblock), q0 + 32);
        const int q = q0 + lane;
        pl = 0;
        cntq = 0;
        if (q < qend) {
          const int32_t* bq = a.bounds + static_cast<int64_t>(q) * (a.nranges + 1);
          pl = bq[r];
          cntq = bq[r + 1] - pl;
        }
        incl = cntq;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        total = __shfl_sync(0xffffffffu, incl, 31);
        cursor = 0;
      }
      if (done) {
        if (lane == 0) {
          t.nc = -1;
          tc::mbar_arrive(&S.tab_full[tb]);
        }
        break;
      }
      const int nc = min(kItemCands, total - cursor);
      int msz[kItemCands / 32], cj[kItemCands / 32], cpos[kItemCands / 32];
      int64_t vb[kItemCands / 32], pb[kItemCands / 32];
#pragma unroll
      for (int i = 0; i < kItemCands / 32; ++i) {
        const int c = lane + 32 * i;
        const int x = cursor + c;  // candidate index of the item: groups of 4 queries in order, and inside a
                                   // group the 4 queries' lists interleaved round-robin, so every tile
                                   // spreads its sets evenly over the 4 TMEM lane quarters (epilogue balance)
        int g = 0;  // group: the smallest g with incl(lane 4g+3) > x
#pragma unroll
        for (int st = 4; st > 0; st >>= 1) {
          const int v = __shfl_sync(0xffffffffu, incl, 4 * (g + st) - 1);
          if (v <= x) g += st;
        }
        g = min(g, 7);
        const int gex = __shfl_sync(0xffffffffu, incl, (4 * g + 31) & 31);  // incl of lane 4g-1 (0 for g = 0)
        int y = x - (g ? gex : 0);
        int cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) cc[u] = __shfl_sync(0xffffffffu, cntq, 4 * g + u);
        const int full = min(min(cc[0], cc[1]), min(cc[2], cc[3]));
        int r = 0, ju = 0;
        if (y < 4 * full) {
          r = y >> 2;
          ju = y & 3;
        } else {
          y -= 4 * full;
          r = full;
          for (;;) {  // round r holds the queries with more than r candidates
            int nr = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) nr += cc[u] > r ? 1 : 0;
            if (y < nr || nr == 0) break;
            y -= nr;
            ++r;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {  // the y-th query (in order) with more than r candidates
            if (cc[u] > r) {
              if (y == 0) {
                ju = u;
                y = -1;
              } else if (y > 0) {
                --y;
              }
            }
          }
        }
        const int j = 4 * g + ju;
        const int plj = __shfl_sync(0xffffffffu, pl, j);
        msz[i] = 0;
        vb[i] = 0;
        pb[i] = 0;
        cj[i] = j;
        cpos[i] = plj + r;
        if (c < nc) {
          const int q = q0 + j;
          const int64_t cid = static_cast<int64_t>(a.cand[static_cast<int64_t>(q) * a.T + cpos[i]]) - a.id_base;
          vb[i] = a.off[cid];
          msz[i] = static_cast<int>(a.off[cid + 1] - vb[i]);
          pb[i] = a.pbase[cid];
          if (msz[i] > kTileRows) {  // exact path: the sentinel (< 0) keeps the set out of K6's k-th select
            a.out_h2[static_cast<int64_t>(q) * a.T + cpos[i]] = kExactSentinel;  // and inside its window
            if (a.out_err) a.out_err[static_cast<int64_t>(q) * a.T + cpos[i]] = 0.0f;
          }
        }
      }
      // tiles: 256 rows, sets whole at 8-aligned columns, and one group of 4 queries (q0 + 4g ..) per tile
      int ntiles = 0, nent = 0, pos = kTileRows, grp = -1;
      unsigned long long rows = 0;
      for (int c = 0; c < nc; ++c) {
        const int m = __shfl_sync(0xffffffffu, msz[c >> 5], c & 31);
        const int j = __shfl_sync(0xffffffffu, cj[c >> 5], c & 31);
        if (m > kTileRows) continue;
        const int mp = (m + 7) & ~7;
        if (pos + ((m + 15) & ~15) > kTileRows || (j >> 2) != grp) {
          if (lane == 0) {
            t.tile_first[ntiles] = nent;
            t.tile_grp[ntiles] = static_cast<int8_t>(j >> 2);
          }
          ++ntiles;
          pos = 0;
          grp = j >> 2;
        }
        if (lane == (c & 31)) {
          t.ent_cand[nent] = cpos[c >> 5];
          t.ent_quarter[nent] = static_cast<int8_t>(j & 3);
          t.ent_col[nent] = static_cast<int16_t>(pos);
          t.ent_m[nent] = static_cast<int16_t>(m);
          t.ent_vbase[nent] = vb[c >> 5];
          t.ent_pbase[nent] = pb[c >> 5];
        }
        ++nent;
        pos += mp;
        rows += static_cast<unsigned long long>(m);
      }
      cursor += nc;
      {  // the item's queries: m_q and first padded row (one load each, lane = query)
        const int q = q0 + lane;
        const bool ok = q < qend;
        const longlong2 mt = ok ? a.qmeta[q] : make_longlong2(0, 0);
        t.gmq[lane] = static_cast<int>(mt.x);
        t.gqr[lane] = mt.y;
      }
      if (lane == 0) {
        t.tile_first[ntiles] = nent;
        t.nc = nc;
        t.q = -1;
        t.c0 = 0;
        t.mq = 32;
        t.rep_rows = 32;
        t.reps = 4;
        t.q0 = 0;
        t.qrow = 0;
        t.gq0 = q0;
        t.gqend = qend;
        t.ntiles = ntiles;
        if (a.rows_counter) atomicAdd(a.rows_counter, rows);
        if (a.prof) atomicAdd(&a.prof[16], static_cast<unsigned long long>(ntiles));  // developer: tiles
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&S.tab_full[tb]);
    }
  } else if (warp == 6) {
    // =========================== item tables (work items, sizes, tile packing) ===========================
    for (uint32_t it = 0;; ++it) {
      const int tb = it & 1;
      ItemTable& t = S.tab[tb];
      PROF_WAIT(0, tc::mbar_wait(&S.tab_empty[tb], ((it >> 1) & 1u) ^ 1u));
      int nc = 0, q = 0, c0 = 0;
      for (;;) {  // next item with at least one candidate
        int item = 0;
        if (lane == 0) item = atomicAdd(a.work_counter, 1);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= a.total_items) {
          nc = -1;
          break;
        }
        q = item / a.items_per_query;
        c0 = (item % a.items_per_query) * kItemCands;
        const int cnt = a.count ? a.count[q] : a.T;
        nc = min(kItemCands, cnt - c0);
        if (nc > 0 && a.qoff[q + 1] - a.qoff[q] > kMaxQ) {  // query rows exceed the M = 128 tile: every
          for (int c = lane; c < nc; c += 32) {                // candidate of this item takes the exact path
            a.out_h2[static_cast<int64_t>(q) * a.T + c0 + c] = kExactSentinel;
            if (a.out_err) a.out_err[static_cast<int64_t>(q) * a.T + c0 + c] = 0.0f;
          }
          continue;
        }
        if (nc > 0) break;
      }
      if (nc < 0) {
        if (lane == 0) {
          t.nc = -1;
          tc::mbar_arrive(&S.tab_full[tb]);
        }
        break;
      }
      const int64_t q0 = a.qoff[q];
      const int mq = static_cast<int>(a.qoff[q + 1] - q0);
      const int rep_rows = mq <= 32 ? 32 : (mq <= 64 ? 64 : 128);
      const int64_t qr = a.qrow[q];
      int msz[kItemCands / 32];
      int64_t vb[kItemCands / 32], pb[kItemCands / 32];
#pragma unroll
      for (int i = 0; i < kItemCands / 32; ++i) {
        const int c = lane + 32 * i;
        msz[i] = 0;
        vb[i] = 0;
        pb[i] = 0;
        if (c < nc) {
          const int64_t cid = static_cast<int64_t>(a.cand[static_cast<int64_t>(q) * a.T + c0 + c]) - a.id_base;
          vb[i] = a.off[cid];
          msz[i] = static_cast<int>(a.off[cid + 1] - vb[i]);
          pb[i] = a.pbase[cid];
          if (msz[i] > x_ncols) {  // exact path: the sentinel (< 0) keeps the set out of K6's k-th select
            a.out_h2[static_cast<int64_t>(q) * a.T + c0 + c] = kExactSentinel;  // and inside its window
            if (a.out_err) a.out_err[static_cast<int64_t>(q) * a.T + c0 + c] = 0.0f;
          }
        }
      }
      float mq2 = 0.0f;
      for (int j = lane; j < kMaxQ; j += 32) {
        t.qn[j] = (j < mq) ? a.qnorm[q0 + j] : 0.0f;
        t.qs2[j] = (j < mq) ? 2.0f * a.qscale[qr + j] : 0.0f;
        mq2 = fmaxf(mq2, t.qn[j]);
      }
      mq2 = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(mq2)));
      if (lane == 0) t.E = a.c1 * sqrtf(mq2) * sqrtf(a.vmax2) + a.c2 * (mq2 + a.vmax2);
      // greedy packing: sets whole inside 256-row tiles at 8-aligned columns
      int ntiles = 0, nent = 0, pos = x_ncols;
      unsigned long long rows = 0;
      for (int c = 0; c < nc; ++c) {
        const int m = __shfl_sync(0xffffffffu, msz[c >> 5], c & 31);
        if (m > x_ncols) continue;
        const int mp = (m + 7) & ~7;
        if (pos + ((m + 15) & ~15) > x_ncols) {  // the epilogue reads 16-column chunks from the set start
          if (lane == 0) t.tile_first[ntiles] = nent;
          ++ntiles;
          pos = 0;
        }
        if (lane == (c & 31)) {
          t.ent_cand[nent] = c;
          t.ent_col[nent] = static_cast<int16_t>(pos);
          t.ent_m[nent] = static_cast<int16_t>(m);
          t.ent_vbase[nent] = vb[c >> 5];
          t.ent_pbase[nent] = pb[c >> 5];
        }
        ++nent;
        pos += mp;
        rows += static_cast<unsigned long long>(m);
      }
      if (lane == 0) {
        t.tile_first[ntiles] = nent;
        t.nc = nc;
        t.q = q;
        t.c0 = c0;
        t.mq = mq;
        t.rep_rows = rep_rows;
        t.reps = kMaxQ / rep_rows;
        t.q0 = q0;
        t.qrow = qr;
        t.ntiles = ntiles;
        if (a.rows_counter) atomicAdd(a.rows_counter, rows);
        if (a.prof) atomicAdd(&a.prof[16], static_cast<unsigned long long>(ntiles));  // developer: tiles
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&S.tab_full[tb]);  // release: the warp's table writes are visible
    }
  } else if (warp == 7) {
    // =========================== tile infos: |v|^2 and scale of every column ===========================
    uint32_t tile_ctr = 0;
    for (uint32_t it = 0;; ++it) {
      const int tb = it & 1;
      const ItemTable& t = S.tab[tb];
      PROF_WAIT(3, tc::mbar_wait(&S.tab_full[tb], (it >> 1) & 1u));
      if (t.nc < 0) break;
      const int ntiles = t.ntiles;
      for (int tile = 0; tile < ntiles; ++tile, ++tile_ctr) {
        const int e0 = t.tile_first[tile], e1 = t.tile_first[tile + 1];
        const int slot = tile_ctr % kInfoSlots;
        TileInfo& inf = S.info[slot];
        PROF_WAIT(2, tc::mbar_wait(&S.info_empty[slot], ((tile_ctr / kInfoSlots) & 1u) ^ 1u));
        float vn8[kTileRows / 32], vs8[kTileRows / 32];
#pragma unroll
        for (int k = 0; k < kTileRows / 32; ++k) {  // lane owns columns lane + 32k: locate the set, load
          const int j = lane + 32 * k;
          vn8[k] = 0.0f;
          vs8[k] = 0.0f;
          if (32 * k >= x_ncols) continue;
          int lo = e0, hi = e1;  // largest e with ent_col[e] <= j
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (t.ent_col[mid] <= j) lo = mid;
            else hi = mid;
          }
          const int r = j - t.ent_col[lo];
          if (r < t.ent_m[lo]) {
            vn8[k] = a.vnorm[t.ent_vbase[lo] + r];
            vs8[k] = a.vscale[t.ent_pbase[lo] + r];
          }
        }
#pragma unroll
        for (int k = 0; k < kTileRows / 32; ++k) {
          if (32 * k >= x_ncols) continue;
          inf.vn[lane + 32 * k] = vn8[k];
          inf.vs[lane + 32 * k] = vs8[k];
        }
        if (lane == 0) {
          inf.first = e0;
          inf.count = e1 - e0;
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.info_full[slot]);
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&S.tab_empty[tb]);
    }
  } else if (warp == 0 || warp >= 12) {
    // =========================== producers: bulk copies ===========================
    // warp 0 arms each stage's barrier and copies the even entries of the tile, warp 12 the odd entries
    // and the query replicas (a bulk copy is issued once per active lane: two warps halve the issue chain)
    const int pw = warp == 0 ? 0 : warp - 11;
    uint32_t stage_ctr = 0;
    for (uint32_t it = 0;; ++it) {
      const int tb = it & 1;
      const ItemTable& t = S.tab[tb];
      PROF_WAIT(7, tc::mbar_wait(&S.tab_full[tb], (it >> 1) & 1u));
      if (t.nc < 0) break;
      const int ntiles = t.ntiles, mq = t.mq, rep_rows = t.rep_rows, reps = t.reps;
      const int64_t qr = t.qrow;
      uint32_t qbytes = static_cast<uint32_t>((mq + 7) & ~7) / 8u * KCS * 1024u;
      uint32_t gbytes[4] = {0u, 0u, 0u, 0u};  // group mode: A bytes / rows of each quarter's query (per tile)
      int64_t gqrow[4] = {0, 0, 0, 0};
      if (x_atmem) {  // the item's query, one super-chunk per stage, once (the MMA warp copies it into TMEM)
        for (int ks = 0; ks < KS; ++ks, ++stage_ctr) {
          const uint32_t st = stage_ctr % NST;
          PROF_WAIT(1, tc::mbar_wait(&S.empty[st], ((stage_ctr / NST) & 1u) ^ 1u));
          if (lane == 0 && pw == 0) {
            mbar_arrive_expect_tx(&S.full[st], qbytes);
            const size_t src = ((static_cast<size_t>(ks) * a.qgroups + (qr >> 3)) * KCS) * 8 * kKChunk;
            bulk_g2s(ring_s + st * a.stage_bytes, a.qhs + src, qbytes, &S.full[st]);
          }
          __syncwarp();
        }
      }
      for (int tile = 0; tile < ntiles; ++tile) {
        const int e0 = t.tile_first[tile], e1 = t.tile_first[tile + 1];
        if (x_group) {  // the tile's 4 queries: q = gq0 + 4 grp + quarter
          const int jb = 4 * t.tile_grp[tile];  // the tile's queries: item slots jb .. jb+3 (table, no global loads)
          qbytes = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            gbytes[j] = static_cast<uint32_t>((t.gmq[jb + j] + 7) & ~7) / 8u * KCS * 1024u;
            gqrow[j] = t.gqr[jb + j];
            qbytes += gbytes[j];
          }
        }
        if (x_prefetch && pw == 0 && tile + 1 < ntiles) {  // warm L2 with the next tile's rows (all K super-chunks)
          const int f0 = t.tile_first[tile + 1], f1 = t.tile_first[tile + 2];
          for (int e = f0 + lane; e < f1; e += 32) {
            const uint32_t nb = static_cast<uint32_t>((t.ent_m[e] + 7) & ~7) / 8u * KCS * 1024u;
            for (int ks = 0; ks < KS; ++ks) {
              const size_t src = ((static_cast<size_t>(ks) * a.pgroups + (t.ent_pbase[e] >> 3)) * KCS) * 8 * kKChunk;
              prefetch_l2(a.hs + src, nb);
              if (three) prefetch_l2(a.ls + src, nb);
            }
          }
        }
        uint32_t bytes = 0;  // B bytes of one piece of one stage
        for (int e = e0 + lane; e < e1; e += 32)
          bytes += (x_tma || x_tail) ? static_cast<uint32_t>(t.ent_m[e]) * KCS * 128u
                         : static_cast<uint32_t>((t.ent_m[e] + 7) & ~7) / 8u * KCS * 1024u;
        bytes = static_cast<uint32_t>(warp_sum(static_cast<int>(bytes)));
        const uint32_t stage_tx = x_atmem ? bytes
                                          : (three ? 2u : 1u) * (bytes + (x_group ? qbytes : static_cast<uint32_t>(reps) * qbytes));
        for (int ks = 0; ks < KS; ++ks, ++stage_ctr) {
          const uint32_t st = stage_ctr % NST;
          PROF_WAIT(1, tc::mbar_wait(&S.empty[st], ((stage_ctr / NST) & 1u) ^ 1u));
          const uint32_t sbase = ring_s + st * a.stage_bytes;
          const uint32_t a_hi = sbase, a_lo = sbase + a.a_bytes;
          const uint32_t b_hi = x_atmem ? sbase : sbase + (three ? 2u : 1u) * a.a_bytes, b_lo = b_hi + a.b_bytes;
          if (lane == 0 && pw == 0) mbar_arrive_expect_tx(&S.full[st], stage_tx);  // (the other warp's copies
          __syncwarp();                                                           // may land first: tx < 0 is legal)
          for (int e = e0 + kProducers * lane + pw; e < e1; e += 32 * kProducers) {
            const int m = t.ent_m[e];
            const int64_t g0 = t.ent_pbase[e] >> 3;
            const size_t src = ((static_cast<size_t>(ks) * a.pgroups + g0) * KCS) * 8 * kKChunk;
            const uint32_t o = static_cast<uint32_t>(t.ent_col[e]) / 8u * KCS * 1024u;
            if (x_tail && KCS == 1) {  // one K-chunk per stage: the set's m rows are one contiguous run
              bulk_g2s(b_hi + o, a.hs + src, static_cast<uint32_t>(m) * 128u, &S.full[st]);
              if (three) bulk_g2s(b_lo + o, a.ls + src, static_cast<uint32_t>(m) * 128u, &S.full[st]);
              continue;
            }
            const bool part = x_tma || x_tail;
            const int full = part ? (m >> 3) : ((m + 7) >> 3), rem = part ? (m & 7) : 0;
            if (full) {  // whole 8-row groups: one contiguous run of full * KCS KB
              const uint32_t nb = static_cast<uint32_t>(full) * KCS * 1024u;
              bulk_g2s(b_hi + o, a.hs + src, nb, &S.full[st]);
              if (three) bulk_g2s(b_lo + o, a.ls + src, nb, &S.full[st]);
            }
            if (rem) {  // the last group's rem real rows, one K-chunk at a time (no padding rows read)
              for (int kc = 0; kc < KCS; ++kc) {
                const uint32_t dst = o + (static_cast<uint32_t>(full) * KCS + kc) * 1024u;
                if (x_tail) {  // plain bulk copies of the rem pre-swizzled rows of each K-chunk
                  const size_t so = src + (static_cast<size_t>(full) * KCS + kc) * 8 * kKChunk;
                  bulk_g2s(b_hi + dst, a.hs + so, static_cast<uint32_t>(rem) * 128u, &S.full[st]);
                  if (three) bulk_g2s(b_lo + dst, a.ls + so, static_cast<uint32_t>(rem) * 128u, &S.full[st]);
                  continue;
                }
                tma_5d(b_hi + dst, &a.tm_hi[rem - 1], 0, 0, kc, static_cast<int>(g0 + full), ks, &S.full[st]);
                if (three) tma_5d(b_lo + dst, &a.tm_lo[rem - 1], 0, 0, kc, static_cast<int>(g0 + full), ks, &S.full[st]);
              }
            }
          }
          if (x_atmem || pw != kProducers - 1) {
          } else if (x_group) {  // group mode: quarter j holds query j's rows (A rows 32j ..)
            if (lane >= 28 && gbytes[lane - 28] > 0) {
              const int j = lane - 28;
              const size_t src = ((static_cast<size_t>(ks) * a.qgroups + (gqrow[j] >> 3)) * KCS) * 8 * kKChunk;
              const uint32_t o = static_cast<uint32_t>(32 * j) / 8u * KCS * 1024u;
              bulk_g2s(a_hi + o, a.qhs + src, gbytes[j], &S.full[st]);
              if (three) bulk_g2s(a_lo + o, a.qls + src, gbytes[j], &S.full[st]);
            }
          } else if (lane >= 32 - reps) {  // query replicas: replica r at A rows r * rep_rows
            const int r = lane - (32 - reps);
            const size_t src = ((static_cast<size_t>(ks) * a.qgroups + (qr >> 3)) * KCS) * 8 * kKChunk;
            const uint32_t o = static_cast<uint32_t>(r * rep_rows) / 8u * KCS * 1024u;
            bulk_g2s(a_hi + o, a.qhs + src, qbytes, &S.full[st]);
            if (three) bulk_g2s(a_lo + o, a.qls + src, qbytes, &S.full[st]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&S.tab_empty[tb]);
    }
  } else if (warp == 1) {
    // =========================== MMA issuer (one thread) ===========================
    uint32_t stage_ctr = 0, tile_ctr = 0;
    const uint32_t idesc = tc::idesc_f16_f32(128, x_ncols);
    for (uint32_t it = 0;; ++it) {
      const int tb = it & 1;
      const ItemTable& t = S.tab[tb];
      PROF_WAIT(4, tc::mbar_wait(&S.tab_full[tb], (it >> 1) & 1u));
      const int nc = t.nc;
      if (nc < 0) break;
      const int ntiles = t.ntiles, rep_rows = t.rep_rows;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&S.tab_empty[tb]);  // the MMA warp needs nothing else from the table
      if (x_atmem) {  // the query into TMEM (the tcgen05 pipe keeps issue order: the previous item's MMAs
                      // have read the old query before these copies overwrite it)
        for (int ks = 0; ks < KS; ++ks, ++stage_ctr) {
          const uint32_t st = stage_ctr % NST;
          PROF_WAIT(6, tc::mbar_wait(&S.full[st], (stage_ctr / NST) & 1u));
          tc::fence_after_sync();
          if (lane == 0) {
            const uint32_t sbase = ring_s + st * a.stage_bytes;
            for (int kc = 0; kc < KCS; ++kc) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {  // 16-byte K slices: 4 TMEM columns each
                const uint32_t col = tmem + a.acol + static_cast<uint32_t>((ks * KCS + kc) * 32 + j * 4);
                const uint64_t d = sw128_desc_sbo(sbase + kc * 1024u + j * 16u, sbo);
                if (rep_rows == 32)
                  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(col), "l"(d) : "memory");
                else if (rep_rows == 64)
                  asm volatile("tcgen05.cp.cta_group::1.64x128b.warpx2::02_13 [%0], %1;" ::"r"(col), "l"(d) : "memory");
                else
                  asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(col), "l"(d) : "memory");
              }
            }
            tc::umma_commit(&S.empty[st]);
          }
          __syncwarp();
        }
      }
      for (int tile = 0; tile < ntiles; ++tile, ++tile_ctr) {
        const uint32_t acc = tile_ctr & 1u;
        PROF_WAIT(5, tc::mbar_wait(&S.tempty[acc], ((tile_ctr >> 1) & 1u) ^ 1u));
        tc::fence_after_sync();
        const uint32_t d_tmem = tmem + acc * x_ncols;
        for (int ks = 0; ks < KS; ++ks, ++stage_ctr) {
          const uint32_t st = stage_ctr % NST;
          PROF_WAIT(6, tc::mbar_wait(&S.full[st], (stage_ctr / NST) & 1u));
          tc::fence_after_sync();
          if (lane == 0) {
            const uint32_t sbase = ring_s + st * a.stage_bytes;
            const uint32_t a_hi = sbase, a_lo = sbase + a.a_bytes;
            const uint32_t b_hi = x_atmem ? sbase : sbase + (three ? 2u : 1u) * a.a_bytes, b_lo = b_hi + a.b_bytes;
            for (int kc = 0; kc < KCS; ++kc) {
#pragma unroll
              for (int kk = 0; kk < kKChunk / 16; ++kk) {
                const uint32_t koff = kc * 1024u + kk * 32u;
                const uint32_t accum = (ks | kc | kk) ? 1u : 0u;
                if (x_atmem) {
                  const uint32_t acol = tmem + a.acol + static_cast<uint32_t>((ks * KCS + kc) * 32 + kk * 8);
                  asm volatile(
                      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
                      "r"(acol), "l"(sw128_desc_sbo(b_hi + koff, sbo)), "r"(idesc), "r"(accum)
                      : "memory");
                  continue;
                }
                tc::umma_bf16(d_tmem, sw128_desc_sbo(a_hi + koff, sbo), sw128_desc_sbo(b_hi + koff, sbo), idesc,
                              accum);
                if (three) {
                  tc::umma_bf16(d_tmem, sw128_desc_sbo(a_hi + koff, sbo), sw128_desc_sbo(b_lo + koff, sbo), idesc, 1u);
                  tc::umma_bf16(d_tmem, sw128_desc_sbo(a_lo + koff, sbo), sw128_desc_sbo(b_hi + koff, sbo), idesc, 1u);
                }
              }
            }
            tc::umma_commit(&S.empty[st]);
            if (ks == KS - 1) tc::umma_commit(&S.tfull[acc]);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // =========================== epilogue (warps 2-5, 8-11) ===========================
    const int ew = warp & 3;                // TMEM lane quarter = query replica rows 32*ew ..
    const int sub = warp >= 8 ? 1 : 0;      // two warps per lane quarter take alternate sets
    uint32_t tile_ctr = 0;
    for (uint32_t it = 0;; ++it) {
      const int tb = it & 1;
      const ItemTable& t = S.tab[tb];
      PROF_WAIT(8, tc::mbar_wait(&S.tab_full[tb], (it >> 1) & 1u));
      const int nc = t.nc;
      if (nc < 0) break;
      const int rep_rows = t.rep_rows, ntiles = t.ntiles;
      const int wpr = rep_rows / 32;          // warps per replica (per sub)
      const int rep = ew / wpr;               // this warp's replica (group mode: its quarter's query)
      const int nrep = 4 / wpr;
      const int qi = (ew % wpr) * 32 + lane;  // query row held by this lane
      int mq = t.mq;
      bool qvalid = qi < mq;
      float qn = qvalid ? t.qn[qi] : 0.0f, qs2 = qvalid ? t.qs2[qi] : 0.0f;
      float* out = a.out_h2 + static_cast<int64_t>(t.q) * a.T + t.c0;
      float* oerr = a.out_err ? a.out_err + static_cast<int64_t>(t.q) * a.T + t.c0 : nullptr;
      const float Eq = t.E, sqE = sqrtf(t.E);
      int gcur = -1;  // group mode: the tile group whose query this warp has loaded
      for (int tile = 0; tile < ntiles; ++tile, ++tile_ctr) {
        const uint32_t acc = tile_ctr & 1u;
        const int slot = tile_ctr % kInfoSlots;
        const TileInfo& inf = S.info[slot];
        PROF_WAIT(9, tc::mbar_wait(&S.tfull[acc], (tile_ctr >> 1) & 1u));
        PROF_WAIT(10, tc::mbar_wait(&S.info_full[slot], (tile_ctr / kInfoSlots) & 1u));
        tc::fence_after_sync();
        const uint32_t tbase = tmem + acc * x_ncols + (static_cast<uint32_t>(ew * 32) << 16);
        const int e0 = inf.first, ne = inf.count;
        if (x_group && t.tile_grp[tile] != gcur) {  // this quarter's query for the tile's group
          gcur = t.tile_grp[tile];
          const int q = t.gq0 + 4 * gcur + ew;
          mq = 0;
          out = nullptr;
          if (q < t.gqend) {  // one level of loads: the packed per-query info (range-major refine)
            const longlong2 mt = a.qmeta[q];
            const float2 pk = a.qpack[static_cast<int64_t>(q) * 32 + lane];
            mq = static_cast<int>(mt.x);
            out = a.out_h2 + static_cast<int64_t>(q) * a.T;
            qn = pk.x;
            qs2 = pk.y;
          }
          qvalid = lane < mq;
        }
        // sets of this tile: replica rep takes sets rep + nrep*k, its two warps (sub) alternate;
        // group mode: quarter ew takes the sets of its query, its two warps alternate
        int gk = 0;
        for (int s = x_group ? 0 : rep + nrep * sub; s < ne; s += x_group ? 1 : 2 * nrep) {
          const int e = e0 + s;
          if (x_group) {
            if (t.ent_quarter[e] != ew) continue;
            if ((gk++ & 1) != sub) continue;
          }
          const int col0 = t.ent_col[e], m = t.ent_m[e];
          float rmin = __int_as_float(0x7f800000);  // per lane (query row): min over the set's columns
          float hv = 0.0f;                          // max over columns of (min over rows)
          float mv = __int_as_float(0x7f800000);    // min over columns of (min over rows): Min metric
          for (int j0 = 0; j0 < m; j0 += 32) {
            uint32_t g[32];
            tc::tmem_ld16(tbase + col0 + j0, *reinterpret_cast<uint32_t(*)[16]>(&g[0]));
            if (j0 + 16 < m) tc::tmem_ld16(tbase + col0 + j0 + 16, *reinterpret_cast<uint32_t(*)[16]>(&g[16]));
            tc::tmem_ld_wait();
#pragma unroll
            for (int j4 = 0; j4 < 32; j4 += 4) {
              if (j0 + j4 < m) {  // warp-uniform
                const float4 vn4 = *reinterpret_cast<const float4*>(&inf.vn[col0 + j0 + j4]);
                const float4 vs4 = *reinterpret_cast<const float4*>(&inf.vs[col0 + j0 + j4]);
                const float vn[4] = {vn4.x, vn4.y, vn4.z, vn4.w}, vs[4] = {vs4.x, vs4.y, vs4.z, vs4.w};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                  const int j = j4 + jj;
                  if (j0 + j < m) {
                    float d2 = __int_as_float(0x7f800000);
                    if (qvalid) d2 = fmaxf(qn + vn[jj] - (qs2 * vs[jj]) * __uint_as_float(g[j]), 0.0f);
                    rmin = fminf(rmin, d2);
                    const uint32_t cmin = __reduce_min_sync(0xffffffffu, __float_as_uint(d2));
                    if (wpr == 1) {
                      hv = fmaxf(hv, __uint_as_float(cmin));
                      mv = fminf(mv, __uint_as_float(cmin));
                    } else if (lane == 0 && METRIC != 1) {
                      atomicMin(&S.cm[rep][col0 + j0 + j], cmin);
                    }
                  }
                }
              }
            }
          }
          if (METRIC == 1) {  // MeanMin: this warp's rows' sum of sqrt(min_v D^2) (fixed butterfly order)
            // and of the per-row error bound: the row minimum a is within E of the exact one b, so
            // |sqrt a - sqrt b| <= min(sqrt E, E / (sqrt a + sqrt max(0, a - E))) (+ the sqrt rounding)
            const float ra = fmaxf(rmin, 0.0f), sa = sqrtf(ra);
            float sq = qvalid ? sa : 0.0f;
            float er = qvalid ? fminf(sqE, Eq / (sa + sqrtf(fmaxf(ra - Eq, 0.0f)))) + 1e-7f * sa : 0.0f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              sq += __shfl_xor_sync(0xffffffffu, sq, o);
              er += __shfl_xor_sync(0xffffffffu, er, o);
            }
            if (wpr == 1) {
              if (lane == 0) {
                out[t.ent_cand[e]] = sq / static_cast<float>(mq);
                oerr[t.ent_cand[e]] = er / static_cast<float>(mq);
              }
            } else if (lane == 0) {
              atomicAdd(reinterpret_cast<float*>(&S.hq[rep][s % kMaxSetsPerTile]), sq);
              atomicAdd(reinterpret_cast<float*>(&S.cm[rep][s % kMaxSetsPerTile]), er);  // (no column minima)
            }
          } else if (METRIC == 2) {  // Min: min over every (query row, set row) of D^2
            if (wpr == 1 && lane == 0) out[t.ent_cand[e]] = mv;
          } else {
            const uint32_t hq = __reduce_max_sync(0xffffffffu, qvalid ? __float_as_uint(rmin) : 0u);
            if (wpr == 1) {
              if (lane == 0) out[t.ent_cand[e]] = fmaxf(__uint_as_float(hq), hv);
            } else if (lane == 0) {
              atomicMax(&S.hq[rep][s % kMaxSetsPerTile], hq);
            }
          }
        }
        // TMEM reads of this tile are done
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.tempty[acc]);
        if (wpr > 1) {  // combine the warps of each replica, then finalize
          tc::named_bar(2, 32 * kEpiWarps);
          if ((ew % wpr) == 0) {  // the replica's first warp (per sub) finalizes its sets
            for (int s = rep + nrep * sub; s < ne; s += 2 * nrep) {
              const int e = e0 + s;
              const int col0 = t.ent_col[e], m = t.ent_m[e];
              if (METRIC == 1) {  // MeanMin: the replica's row sums (value, error bound)
                if (lane == 0) {
                  const int sl = s % kMaxSetsPerTile;
                  out[t.ent_cand[e]] = __uint_as_float(S.hq[rep][sl]) / static_cast<float>(mq);
                  oerr[t.ent_cand[e]] = __uint_as_float(S.cm[rep][sl]) / static_cast<float>(mq);
                  S.hq[rep][sl] = 0u;
                  S.cm[rep][sl] = 0u;
                }
                continue;
              }
              float hv = 0.0f, mv = __int_as_float(0x7f800000);
              for (int j = lane; j < m; j += 32) {
                hv = fmaxf(hv, __uint_as_float(S.cm[rep][col0 + j]));
                mv = fminf(mv, __uint_as_float(S.cm[rep][col0 + j]));
                S.cm[rep][col0 + j] = 0x7f800000u;
              }
              hv = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(hv)));
              mv = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(mv)));
              if (lane == 0) {
                const uint32_t acc_hq = S.hq[rep][s % kMaxSetsPerTile];
                out[t.ent_cand[e]] = METRIC == 1   ? __uint_as_float(acc_hq) / static_cast<float>(mq)
                                     : METRIC == 2 ? mv
                                                     : fmaxf(__uint_as_float(acc_hq), hv);
                S.hq[rep][s % kMaxSetsPerTile] = 0u;
              }
            }
          }
          tc::named_bar(2, 32 * kEpiWarps);
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.info_empty[slot]);
      }
      __syncwarp();
      tc::named_bar(3, 32 * kEpiWarps);  // every epilogue warp is done with this item's table
      if (tid == 64) tc::mbar_arrive(&S.tab_empty[tb]);
    }
  }
  if (a.prof && lane == 0 && (warp <= 2 || warp == 6 || warp == 7))
    atomicAdd(&a.prof[warp <= 2 ? 12 + warp : (warp == 6 ? 15 : 11)], (unsigned long long)(clock64() - t_role0));
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, 512);
  }
}

// bounds[q][r] = first position of cand[q] whose (ascending) id lies in range r or later (r = 0..R);
// bounds[q][R] = count[q].  Warp per query.
__global__ void range_bounds_kernel(const int32_t* __restrict__ cand, const int32_t* __restrict__ count, int T, int nq,
                                    int64_t id_base, int64_t range_sets, int R, int32_t* __restrict__ bounds) {
  const int lane = threadIdx.x & 31;
  for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < nq; q += (gridDim.x * blockDim.x) >> 5) {
    const int cnt = count ? count[q] : T;
    const int32_t* row = cand + static_cast<int64_t>(q) * T;
    int32_t* bq = bounds + static_cast<int64_t>(q) * (R + 1);
    for (int p = lane; p <= cnt; p += 32) {
      const int rp = p < cnt ? static_cast<int>((row[p] - id_base) / range_sets) : R;
      const int rprev = p == 0 ? -1 : static_cast<int>((row[p - 1] - id_base) / range_sets);
      for (int r = rprev + 1; r <= rp && r <= R; ++r) bq[r] = p;
    }
  }
}

// packed per-query info of the range-major refine: (|q_i|^2, 2 s_i) per row, (m_q, first padded row)
__global__ void query_pack_kernel(const int64_t* __restrict__ qoff, const int64_t* __restrict__ qrow,
                                  const float* __restrict__ qnorm, const float* __restrict__ qscale, int nq,
                                  float2* __restrict__ qpack, longlong2* __restrict__ qmeta) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nq * 32; t += gridDim.x * blockDim.x) {
    const int q = t >> 5, i = t & 31;
    const int64_t q0 = qoff[q];
    const int mq = static_cast<int>(qoff[q + 1] - q0);
    qpack[t] = i < mq ? make_float2(qnorm[q0 + i], 2.0f * qscale[qrow[q] + i]) : make_float2(0.0f, 0.0f);
    if (i == 0) qmeta[q] = make_longlong2(mq, qrow[q]);
  }
}

// Group-mode plan: database sets per range and the number of ranges (0 = query-major).
// A range holds ~9 candidates of every query and its rows fit a 40 MB share of L2.
int64_t refine_range_sets(int64_t n_local, int64_t prows, int dpad, int T) {
  if (n_local <= 0) return 0;
  const double set_bytes = static_cast<double>(prows) / static_cast<double>(n_local) * dpad * 2.0;
  int64_t rs = static_cast<int64_t>(static_cast<double>(n_local) * 9.0 / T);
  const int64_t cap = static_cast<int64_t>(40.0 * (1 << 20) / set_bytes);
  if (rs > cap) rs = cap;
  if (const char* r = getenv("BVSS_REFINE_RANGE")) rs = atoll(r);  // developer switch
  if (rs < 64) rs = 64;
  if (rs > n_local) rs = n_local;
  return rs;
}

int refine_kcs(int dpad) {
  static const int forced = [] {  // developer switch: K-chunks per stage (1, 2 or 3; must divide dpad/64)
    const char* e = getenv("BVSS_REFINE_KCS");
    return e ? atoi(e) : 0;
  }();
  if (forced > 0 && (dpad / kKChunk) % forced == 0) return forced;
  return (dpad / kKChunk) % 2 == 0 ? 2 : 1;
}

size_t refine_smem_bytes(int terms, int KCS, int atmem, int ncols, int& stages, uint32_t& stage_bytes) {
  const uint32_t a_bytes = 128u * KCS * 128u, b_bytes = static_cast<uint32_t>(ncols) * KCS * 128u;
  stage_bytes = atmem ? b_bytes : (terms == 3 ? 2u : 1u) * (a_bytes + b_bytes);
  const size_t ctrl = (sizeof(RefineCtl) + 127) & ~size_t(127);  // static __shared__
  const size_t budget = 227 * 1024 - 1024 - ctrl;
  stages = static_cast<int>(budget / stage_bytes);
  if (stages > kMaxStages) stages = kMaxStages;
  return static_cast<size_t>(stages) * stage_bytes + 1024;
}

int launch_refine_tc(const __half* hs, const __half* ls, const float* vscale, int64_t prows, const int64_t* pbase,
                     const float* vnorm, const int64_t* off, int dpad, const __half* qhs, const __half* qls,
                     const float* qscale, int64_t qrows, const int64_t* qrow, const float* qnorm, const int64_t* qoff,
                     int max_mq, const int32_t* cand, const int32_t* count, int T, int nq, int64_t id_base,
                     float* out_h2, int terms, int* work_counter, unsigned long long* rows_counter, int num_sms,
                     int64_t n_local, int32_t* bounds, int metric, float* out_err, float c1, float c2, float vmax2,
                     cudaStream_t st) {
  if (nq <= 0 || T <= 0) return BVSS_OK;
  // query sets > kMaxQ rows are routed per query to the exact path (item table warp)
  if (dpad % kKChunk) BVSS_FAIL(BVSS_EINVAL, "dpad must be a multiple of 64");
  RefineArgs a;
  a.hs = hs; a.ls = ls; a.vscale = vscale; a.pgroups = prows / 8; a.pbase = pbase; a.vnorm = vnorm; a.off = off;
  a.KC = dpad / kKChunk;
  a.KCS = refine_kcs(dpad);
  a.qhs = qhs; a.qls = qls; a.qscale = qscale; a.qgroups = qrows / 8; a.qrow = qrow; a.qnorm = qnorm; a.qoff = qoff;
  a.cand = cand; a.count = count; a.T = T; a.nq = nq; a.id_base = id_base; a.out_h2 = out_h2;
  a.terms = terms == 3 ? 3 : 1;
  a.metric = metric;
  a.out_err = out_err;
  a.c1 = c1;
  a.c2 = c2;
  a.vmax2 = vmax2;
  if (metric == 1 && !out_err) BVSS_FAIL(BVSS_EINVAL, "MeanMin refine needs the error-bound output");
  a.items_per_query = ceil_div(T, kItemCands);
  a.total_items = a.items_per_query * nq;
  a.work_counter = work_counter;
  a.rows_counter = rows_counter;
  {
    const char* e = getenv("BVSS_REFINE_PREFETCH");
    a.prefetch = e ? atoi(e) : 0;
  }
  static unsigned long long* prof = nullptr;
  a.prof = nullptr;
  if (getenv("BVSS_REFINE_PROF")) {
    if (!prof) cudaMalloc(&prof, 17 * sizeof(unsigned long long));
    cudaMemsetAsync(prof, 0, 17 * sizeof(unsigned long long), st);
    a.prof = prof;
  }
  a.bounds = nullptr;
  // group mode: needs every query set within one TMEM lane quarter (m_q <= 32) and
  // ascending candidate lists (n_local > 0 and bounds != null from the caller)
  a.group = 0;
  {
    // off by default: measured 8x less DRAM traffic but 1.45x slower per tile than query-major (r01 notes)
    const char* e = getenv("BVSS_REFINE_GROUP");  // developer switch: 1 = range-major group items
    const int want = e ? atoi(e) : 0;
    const int64_t rs = refine_range_sets(n_local, prows, dpad, T);
    if (want && metric == 0 && max_mq <= 32 && nq >= 16 && rs > 0 && bounds) {
      const double qbytes = 32.0 * dpad * 2.0;                    // A rows of one query (upper bound)
      int qb = static_cast<int>(60.0 * (1 << 20) / qbytes);      // query rows of a block stay in L2
      if (const char* b = getenv("BVSS_REFINE_QBLOCK")) qb = atoi(b);
      qb = qb < 32 ? 32 : qb;
      qb = (qb + 31) & ~31;
      if (qb > ((nq + 31) & ~31)) qb = (nq + 31) & ~31;
      const int64_t nranges = (n_local + rs - 1) / rs;
      const int64_t nblocks = (nq + qb - 1) / qb;
      const int64_t items = nblocks * nranges * (qb / 32);
      if (items < (1ll << 31)) {
        a.group = 1;
        a.qblock = qb;
        a.range_sets = rs;
        a.nranges = static_cast<int>(nranges);
        a.n_local = n_local;
        a.total_items = static_cast<int>(items);
        a.bounds = bounds;
        // the caller's buffer: bounds [nq][nranges+1] int32, then qmeta [nq] (16 B), then qpack [nq][32] (8 B)
        const size_t boff = ((static_cast<size_t>(nq) * (nranges + 1) * 4) + 15) & ~size_t(15);
        longlong2* qmeta = reinterpret_cast<longlong2*>(reinterpret_cast<uint8_t*>(bounds) + boff);
        float2* qpack = reinterpret_cast<float2*>(qmeta + nq);
        a.qmeta = qmeta;
        a.qpack = qpack;
        range_bounds_kernel<<<num_sms * 8, 256, 0, st>>>(cand, count, T, nq, id_base, rs, a.nranges, bounds);
        BVSS_TRY(post_launch("range_bounds_kernel", st));
        query_pack_kernel<<<num_sms * 4, 256, 0, st>>>(qoff, qrow, qnorm, qscale, nq, qpack, qmeta);
        BVSS_TRY(post_launch("query_pack_kernel", st));
      }
    }
  }
  {  // TMA maps for the partial last group of every set (h = 1..8 rows)
    const char* e = getenv("BVSS_REFINE_TMA");  // developer switch: 0 = copy whole padded groups
    a.tma = e ? atoi(e) : 0;
    const char* f = getenv("BVSS_REFINE_TAIL");
    a.tail = f ? atoi(f) : 0;
    if (a.tail) a.tma = 0;
  }
  if (a.tma) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      BVSS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
      if (!fn || q != cudaDriverEntryPointSuccess) BVSS_FAIL(BVSS_ECUDA, "cuTensorMapEncodeTiled unavailable");
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[5] = {64, 8, static_cast<cuuint64_t>(a.KCS), static_cast<cuuint64_t>(a.pgroups),
                                static_cast<cuuint64_t>(a.KC / a.KCS)};
    const cuuint64_t strides[4] = {128, 1024, static_cast<cuuint64_t>(a.KCS) * 1024,
                                   static_cast<cuuint64_t>(a.pgroups) * a.KCS * 1024};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    for (int h = 1; h <= 8; ++h) {
      const cuuint32_t box[5] = {64, static_cast<cuuint32_t>(h), 1, 1, 1};
      for (int piece = 0; piece < (a.terms == 3 ? 2 : 1); ++piece) {
        CUresult r = encode(piece ? &a.tm_lo[h - 1] : &a.tm_hi[h - 1], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5,
                            const_cast<__half*>(piece ? ls : hs), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) BVSS_FAIL(BVSS_ECUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
      }
    }
  }
  // A in TMEM: one term, query-major, and TMEM room for the query (dpad/2 columns)
  // next to two accumulators of at least 128 columns
  a.atmem = 0;
  a.ncols = kTileRows;
  a.acol = 0;
  {
    // developer switch BVSS_REFINE_ATMEM=1, off by default: measured slower (67.6 vs 53.9 ms at cfg3,
    // tools/ab_env.py): a tcgen05.mma costs ~200 cycles whatever N (tools/microbench_umma.cu), so the
    // narrower N = 160 tiles the TMEM budget leaves cost 1.6x the MMA time per candidate row
    const char* e = getenv("BVSS_REFINE_ATMEM");
    const int want = e ? atoi(e) : 0;
    const int ncols = ((512 - dpad / 2) / 2) & ~15;
    if (want && a.terms == 1 && !a.group && !a.tma && !a.tail && ncols >= 128) {
      a.atmem = 1;
      a.ncols = ncols < kTileRows ? ncols : kTileRows;
      a.acol = static_cast<uint32_t>(2 * a.ncols);
    }
    if (const char* f = getenv("BVSS_REFINE_NCOLS")) {  // developer switch: tile width (multiple of 16)
      const int nf = atoi(f);
      if (nf >= 32 && nf % 16 == 0 && nf <= a.ncols) a.ncols = nf;
      if (a.atmem) a.acol = 512u - static_cast<uint32_t>(dpad / 2);
    }
  }
  int stages;
  uint32_t stage_bytes;
  const size_t smem = refine_smem_bytes(a.terms, a.KCS, a.atmem, a.ncols, stages, stage_bytes);
  if (stages < 1) BVSS_FAIL(BVSS_EUNSUPPORTED, "refine stage does not fit shared memory");
  a.stages = stages;
  a.stage_bytes = stage_bytes;
  a.a_bytes = 128u * a.KCS * 128u;
  a.b_bytes = static_cast<uint32_t>(a.ncols) * a.KCS * 128u;
  BVSS_CUDA(cudaMemsetAsync(work_counter, 0, sizeof(int), st));
  const int grid = a.total_items < num_sms ? a.total_items : num_sms;
  const bool exper = a.atmem || a.tail || a.tma || a.group || a.prefetch || a.ncols != kTileRows || a.terms == 3;
  auto kfn = exper ? (metric == 1 ? refine_tc_kernel<1, true> : metric == 2 ? refine_tc_kernel<2, true> : refine_tc_kernel<0, true>)
                   : (metric == 1 ? refine_tc_kernel<1, false> : metric == 2 ? refine_tc_kernel<2, false> : refine_tc_kernel<0, false>);
  BVSS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kfn<<<grid, kRefineThreads, smem, st>>>(a);
  BVSS_TRY(post_launch(__func__, st));
  if (a.prof) {  // developer instrumentation: per-CTA average Mcycles per role
    unsigned long long h[17];
    cudaMemcpyAsync(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const double g = grid;
    fprintf(stderr,
            "[refine prof] per CTA Mcycles: copy %.2f (tab %.2f, empty %.2f) | table %.2f (tab_empty %.2f) | info %.2f "
            "(tab %.2f, info_empty %.2f) | mma %.2f (tab %.2f, tempty %.2f, full %.2f) | epilogue %.2f (tab %.2f, "
            "tfull %.2f, info %.2f)\n",
            h[12] / g / 1e6, h[7] / g / 1e6, h[1] / g / 1e6, h[15] / g / 1e6, h[0] / g / 1e6, h[11] / g / 1e6, h[3] / g / 1e6, h[2] / g / 1e6, h[13] / g / 1e6, h[4] / g / 1e6, h[5] / g / 1e6,
            h[6] / g / 1e6, h[14] / g / 1e6, h[8] / g / 1e6 / kEpiWarps, h[9] / g / 1e6 / kEpiWarps, h[10] / g / 1e6 / kEpiWarps);
    fprintf(stderr, "[refine prof] tiles %llu (group mode %d)\n", h[16], a.group);
  }
  return BVSS_OK;
}

}  // namespace bvss
