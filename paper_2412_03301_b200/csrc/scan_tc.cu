// scan_tc.cu — K3 on the 5th-generation tensor cores: the filter scan of Alg 6
// lines 10-13 as an exact GEMM between query sketches and database
// sketches, accumulated in TMEM.
//
//   binary : popc(S_Q AND S_i) = sum_j b_Q[j] b_i[j].  Every sketch bit is an
//            e2m1 (FP4) element, 1.0 or 0.0, and the product runs as
//            tcgen05.mma kind::mxf4 with all block scales = 1.0 (ue8m0 127):
//            products are 0/1 and the fp32 sums are integers <= m < 2^24, so
//            the count is exact.  Hamming = p_Q + p_i - 2 popc(AND)   (reading R1)
//   count  : <C_Q, C_i> = sum_j C_Q[j] C_i[j] on the uint8 counters, kind::i8
//            (u8 x u8 -> s32); L2^2 = |C_Q|^2 + |C_i|^2 - 2 <C_Q, C_i>  (reading R2)
// Both are exact, so the keys are bit-identical to the SIMT scan (scan.cu) and
// to the oracle.  Measured on B200 (tools/microbench_scan_mma.cu): kind::mxf4
// M=128 N=240 K=64 issues every ~154 cycles (12.8k MAC/clk/SM), kind::i8 M=128
// N=256 K=32 every ~161 cycles (6.5k MAC/clk/SM).
//
// Operands use the canonical no-swizzle K-major layout: per 16-byte K unit u a
// [rows][16 B] block (core matrices of 8 rows x 16 B), LBO = rows x 16 B
// between units, SBO = 128 B between 8-row groups.  The index stores the
// database operand in exactly this layout ([units][n][16 B]: the FP4 expansion
// of the binary sketches, made once at build time, or the count sketches), so
// every tile arrives by plain contiguous cp.async.bulk copies and no SM time is
// spent on bit expansion.
//
// A = a tile of 128 query sketches (M = 128, one TMEM lane per query), B = kN
// database sets (N = 240 FP4 / 256 i8), 128 bytes of K per stage (4 MMAs).  One
// operand is STATIONARY in shared memory (scan_tc_mode): by default the database
// tile (MODE_BRES: query tiles stream through the stage ring from L2), else the
// query tile (MODE_ARES), else both stream (MODE_STREAM).  The (query tile,
// database tile) pairs are ordered by the stationary operand and split into
// equal contiguous ranges, one per persistent CTA, so a CTA reloads its
// stationary tile at most a few times.
//
// Because a TMEM lane is a query, the epilogue thread owns one query: its mass
// p_Q and threshold tau_Q live in registers and the per-value work is one FFMA
// (IMAD for i8) and one compare: p_i - 2 acc <= tau_Q - p_Q (database masses
// come from a shared-memory slot the producer fills per tile; all values are
// exact integers in fp32).  Emit mode appends (id, key)
// for key <= tau_Q: a first pass over the tile's columns builds per-column pass
// bits, one atomic per (thread, tile) reserves the buffer range, and a second
// TMEM pass writes the entries.
//
// CTA = 14 warps: warp 0 producer (query tile, stage copies, database masses),
// warp 1 TMEM owner + MMA issuer, warps 2-13 epilogue (three per TMEM lane
// quarter, 96 columns each).  Double-buffered TMEM accumulators (2 x kN columns; FP4 keeps its
// block scales in the last 32 columns).
#include <cstdlib>
#include <type_traits>

#include "tc.cuh"

namespace bvss {

constexpr int kScanM = 128;        // queries per tile (MMA M, TMEM lanes)
constexpr int kScanStageB = 128;   // bytes of K per row per stage (8 units of 16 B, 4 MMAs)
constexpr int kScanThreads = 448;  // 14 warps: 128 registers per thread
constexpr int kScanEpiWarps = 12;
constexpr int kScanEpiCols = 96;  // columns per epilogue warp (three per TMEM lane quarter)
constexpr int kScanSmemBudget = 220 * 1024;
constexpr int kScanMaxStages = 8;
constexpr uint32_t kScaleOne = 0x7F7F7F7Fu;  // four ue8m0 scale factors = 2^0
constexpr int kMassSlots = 4;  // mass slots: the producer runs up to 4 tiles ahead of the epilogue

struct ScanArgs {
  const uint4* S;              // DB operand [U][n_stride][16 B] (FP4 expansion or u8 counters)
  const int32_t* massS;        // [n]
  int64_t n, n_stride;
  const uint4* Qx;             // query operand [qpad/128][U][128 rows][16 B] (query-tile-major)
  const int32_t* massQ;        // [nq]
  int nq, qpad;
  int U;                       // 16-byte K units per row
  void* keys;                  // [nq][key_stride] uint16 (binary) / uint32 (count)
  int64_t key_stride;
  int n_tiles, q_tiles;
  // threshold-emit mode (EMIT = true): keys <= tau[q] are appended to per-query buffers
  const uint32_t* tau;     // [nq]
  int32_t* cnt;            // [nq] entries emitted (may exceed cap: overflow)
  int32_t* buf_id;         // [nq][cap] set ids (+ id_base)
  uint32_t* buf_key;       // [nq][cap] keys
  int cap;
  int64_t id_base;
  int dbg;  // developer switch (env BVSS_SCAN_DBG=1): the epilogue only releases the accumulators
};

template <int KS, int N>
struct ScanCtl {
  uint64_t full[KS];
  uint64_t empty[KS];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint64_t afull, aempty;
  uint64_t mfull[kMassSlots], mempty[kMassSlots];  // database masses of a tile (producer -> epilogue)
  uint32_t tmem_base;
  __align__(16) uint32_t mass[kMassSlots][256];  // FP4: float bits; i8: int
  uint32_t emit_mask[kScanEpiWarps][kScanEpiCols / 32][32];  // emit pass-1 bits [warp][chunk][lane]
};

__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// no-swizzle K-major descriptor: LBO = stride between 16-byte K units, SBO = stride between 8-row groups
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;  // version (sm_100)
  return d;                              // layout type 0 = SWIZZLE_NONE
}
// instruction descriptors: kind::i8 (u8 x u8 -> s32) and kind::mxf4 (e2m1 x e2m1, ue8m0 scales -> f32)
__host__ __device__ __forceinline__ uint32_t idesc_u8_s32(int M, int N) {
  return (2u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}
__host__ __device__ __forceinline__ uint32_t idesc_mxf4(int M, int N) {
  return (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (1u << 23) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void umma_u8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_fp4(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate, uint32_t sfa, uint32_t sfb) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
      : "memory");
}
// 8 sketch bits -> 8 e2m1 nibbles (bit e -> nibble e: 0x2 = 1.0 or 0x0)
__host__ __device__ __forceinline__ uint32_t bits8_to_fp4(uint32_t b) {
  uint32_t x = b & 0xFFu;
  x = (x | (x << 12)) & 0x000F000Fu;
  x = (x | (x << 6)) & 0x03030303u;
  x = (x | (x << 3)) & 0x11111111u;
  return x << 1;
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  tc::tmem_ld16(taddr, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
  tc::tmem_ld16(taddr + 16, *reinterpret_cast<uint32_t(*)[16]>(&r[16]));
}

// Work split: the (query tile, database tile) pairs are ordered by the
// STATIONARY operand -- query-tile-major when the query tile stays in smem
// (MODE_ARES / MODE_STREAM), database-tile-major when the database tile does
// (MODE_BRES) -- and cut into gridDim.x equal contiguous ranges, one per CTA
// (exact balance).  A "run" is a maximal stretch of a CTA's range with the same
// stationary tile; the stationary operand is loaded once per run.
enum { MODE_ARES = 0, MODE_STREAM = 1, MODE_BRES = 2 };

struct TileSeq {
  int64_t f, f0, f1;
  int inner;
  bool dbmajor;
  __device__ TileSeq(const ScanArgs& a, bool db_major) {
    const int64_t W = static_cast<int64_t>(a.q_tiles) * a.n_tiles;
    f0 = f = W * blockIdx.x / gridDim.x;
    f1 = W * (blockIdx.x + 1) / gridDim.x;
    inner = db_major ? a.q_tiles : a.n_tiles;
    dbmajor = db_major;
  }
  // next tile (qt, t); first / last = first / last tile of its run
  __device__ bool next(int& qt, int& t, bool& first, bool& last) {
    if (f >= f1) return false;
    const int64_t key = f / inner;
    const int pos = static_cast<int>(f - key * inner);
    qt = dbmajor ? pos : static_cast<int>(key);
    t = dbmajor ? static_cast<int>(key) : pos;
    first = pos == 0 || f == f0;
    ++f;
    last = f >= f1 || (f % inner) == 0;
    return true;
  }
};

// FP4 = binary sketches (kind::mxf4, N = 240, uint16 keys); else count sketches (kind::i8, N = 256, uint32 keys)
template <bool FP4, bool EMIT, int MODE, int KS>
__global__ void __launch_bounds__(kScanThreads, 1) scan_tc_kernel(ScanArgs a) {
  using KeyT = typename std::conditional<FP4, uint16_t, uint32_t>::type;
  constexpr int N = FP4 ? 240 : 256;
  constexpr bool ARES = MODE == MODE_ARES, BRES = MODE == MODE_BRES;
  constexpr uint32_t kBStage = BRES ? 0u : N * kScanStageB;
  constexpr uint32_t kAStage = ARES ? 0u : kScanM * kScanStageB;
  constexpr uint32_t kStage = kAStage + kBStage;
  constexpr uint32_t kAcc = FP4 ? 240u : 256u;  // accumulator buffer b at columns [b kAcc, b kAcc + N)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ ScanCtl<KS, N> S;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t res = smem_u32(base);  // the resident (stationary) tile
  const uint32_t ring =
      res + (ARES ? static_cast<uint32_t>(kScanM) * a.U * 16u : (BRES ? static_cast<uint32_t>(N) * a.U * 16u : 0u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KC = a.U / 8;  // stages per tile

  if (tid == 0) {
    for (int s = 0; s < KS; ++s) {
      tc::mbar_init(&S.full[s], 1);
      tc::mbar_init(&S.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&S.tfull[b], 1);
      tc::mbar_init(&S.tempty[b], kScanEpiWarps);
    }
    for (int b = 0; b < kMassSlots; ++b) {
      tc::mbar_init(&S.mfull[b], 32);
      tc::mbar_init(&S.mempty[b], kScanEpiWarps);
    }
    tc::mbar_init(&S.afull, 1);
    tc::mbar_init(&S.aempty, 1);
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(&S.tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = S.tmem_base;
  if (FP4 && warp >= 2 && warp < 6) {  // block scales = 1.0 in columns [480, 512) of every lane
    const uint32_t taddr = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 480u;
#pragma unroll 1
    for (int c = 0; c < 32; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr + c), "r"(kScaleOne) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();

  if (warp == 0) {
    // ------------------------------------------------------------- producer
    uint32_t sc = 0, rc = 0, tc_ = 0;
    TileSeq seq(a, BRES);
    int qt, t;
    bool first, last;
    while (seq.next(qt, t, first, last)) {
      const int64_t i0 = static_cast<int64_t>(t) * N;
      const int rows = static_cast<int>(a.n - i0 < N ? a.n - i0 : N);
      if (first && !(MODE == MODE_STREAM)) {  // the stationary tile of this run: U units of [rows][16 B]
        tc::mbar_wait(&S.aempty, (rc & 1u) ^ 1u);
        const uint32_t rrows = ARES ? kScanM : N;
        if (lane == 0) arrive_expect_tx(&S.afull, (ARES ? kScanM : rows) * a.U * 16u);
        __syncwarp();
        if (ARES) {  // the query tile is one contiguous run of U x 2 KB (query-tile-major Qx)
          if (lane == 0)
            bulk_copy(res, a.Qx + static_cast<int64_t>(qt) * a.U * kScanM, static_cast<uint32_t>(a.U) * kScanM * 16u,
                      &S.afull);
        } else {
          for (int uu = lane; uu < a.U; uu += 32)
            bulk_copy(res + uu * (rrows * 16u), a.S + static_cast<int64_t>(uu) * a.n_stride + i0,
                      static_cast<uint32_t>(rows) * 16u, &S.afull);
        }
        ++rc;
      }
      {  // masses of the tile's sets -> smem slot tc_ % 4 (columns past n get a huge mass: never selected)
        const uint32_t slot = tc_ % kMassSlots;
        tc::mbar_wait(&S.mempty[slot], ((tc_ / kMassSlots) & 1u) ^ 1u);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = lane * 8 + j;
          const int32_t mv = (c < rows) ? __ldg(a.massS + i0 + c) : 0x40000000;  // huge: never selected
          S.mass[slot][c] = FP4 ? __float_as_uint(static_cast<float>(mv)) : static_cast<uint32_t>(mv);
        }
        tc::mbar_arrive(&S.mfull[slot]);
      }
      for (int kc = 0; kc < KC; ++kc, ++sc) {
        const int st = sc % KS;
        tc::mbar_wait(&S.empty[st], ((sc / KS) & 1u) ^ 1u);
        const uint32_t sa = ring + st * kStage, sb = sa + kAStage;
        if (lane == 0) arrive_expect_tx(&S.full[st], kAStage + (BRES ? 0u : 8u * rows * 16u));
        __syncwarp();
        if (!BRES && lane < 8) {  // DB units 8kc .. 8kc+7
          const int uu = 8 * kc + lane;
          bulk_copy(sb + lane * (N * 16u), a.S + static_cast<int64_t>(uu) * a.n_stride + i0,
                    static_cast<uint32_t>(rows) * 16u, &S.full[st]);
        } else if (!ARES && lane == 8) {  // streamed A: units 8kc .. 8kc+7 of the query tile, one 16 KB run
          bulk_copy(sa, a.Qx + (static_cast<int64_t>(qt) * a.U + 8 * kc) * kScanM, 8u * kScanM * 16u, &S.full[st]);
        }
      }
      ++tc_;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = FP4 ? idesc_mxf4(kScanM, N) : idesc_u8_s32(kScanM, N);
    uint32_t sc = 0, tc_ = 0, rc = 0;
    TileSeq seq(a, BRES);
    int qt, t;
    bool first, last;
    while (seq.next(qt, t, first, last)) {
      if (first && MODE != MODE_STREAM) {
        tc::mbar_wait(&S.afull, rc & 1u);
        tc::fence_after_sync();
      }
      const uint32_t acc = tc_ & 1u;
      tc::mbar_wait(&S.tempty[acc], ((tc_ >> 1) & 1u) ^ 1u);
      tc::fence_after_sync();
      const uint32_t d = tmem + acc * kAcc;
      for (int kc = 0; kc < KC; ++kc, ++sc) {
        const int st = sc % KS;
        tc::mbar_wait(&S.full[st], (sc / KS) & 1u);
        tc::fence_after_sync();
        if (lane == 0) {
          const uint32_t sa = ring + st * kStage, sb = sa + kAStage;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // 32 bytes of K (2 units) per instruction
            const uint32_t u = 8 * kc + 2 * kk;
            const uint64_t ad = ARES ? kmajor_desc(res + u * (kScanM * 16u), kScanM * 16u, 128u)
                                     : kmajor_desc(sa + 2 * kk * (kScanM * 16u), kScanM * 16u, 128u);
            const uint64_t bd = BRES ? kmajor_desc(res + u * (N * 16u), N * 16u, 128u)
                                     : kmajor_desc(sb + 2 * kk * (N * 16u), N * 16u, 128u);
            const uint32_t accum = (kc | kk) ? 1u : 0u;
            if (FP4) umma_fp4(d, ad, bd, idesc, accum, tmem + 480u, tmem + 496u);
            else umma_u8(d, ad, bd, idesc, accum);
          }
          tc::umma_commit(&S.empty[st]);
          if (kc == KC - 1) {
            tc::umma_commit(&S.tfull[acc]);
            if (last && MODE != MODE_STREAM) tc::umma_commit(&S.aempty);  // the stationary tile may be replaced
          }
        }
        __syncwarp();
      }
      if (first && MODE != MODE_STREAM) ++rc;
      ++tc_;
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2-13)
    const int quarter = warp & 3;           // TMEM lane quarter this warp may access
    const int part = (warp - 2) >> 2;       // columns [cb, ce): [0, 96), [96, 192), [192, N)
    const int cb = part * kScanEpiCols, ce = min(N, cb + kScanEpiCols);
    KeyT* keys = static_cast<KeyT*>(a.keys);
    uint32_t tc_ = 0;
    TileSeq seq(a, BRES);
    int qt, t;
    bool first, last;
    int qcur = -1;
    int32_t pq = 0, lim = 0;
    float limf = 0.0f, pqf = 0.0f;
    bool qok = false;
    int q = 0;
    while (seq.next(qt, t, first, last)) {
      if (qt != qcur) {
        qcur = qt;
        q = qt * kScanM + quarter * 32 + lane;
        qok = q < a.nq;
        pq = qok ? __ldg(a.massQ + q) : 0;
        // key <= tau  <=>  p_i - 2 acc <= tau - p_Q   (keys are exact integers < 2^24 (FP4) / 2^31 (i8))
        lim = EMIT ? (qok ? static_cast<int32_t>(__ldg(a.tau + q)) - pq : -0x40000000) : 0;
        limf = static_cast<float>(lim);
        pqf = static_cast<float>(pq);
      }
      {
        const uint32_t acc = tc_ & 1u;
        const int64_t i0 = static_cast<int64_t>(t) * N;
        const uint32_t ms = tc_ % kMassSlots;  // mass slot of this tile
        tc::mbar_wait(&S.mfull[ms], (tc_ / kMassSlots) & 1u);
        tc::mbar_wait(&S.tfull[acc], (tc_ >> 1) & 1u);
        tc::fence_after_sync();
        const uint32_t tbase = tmem + acc * kAcc + (static_cast<uint32_t>(quarter * 32) << 16);
        // masses: float (FP4: the accumulator is an exact integer-valued f32) or int (i8: s32 accumulator)
        auto load_mass = [&](int c0, uint32_t (&pi)[32]) {
          const uint4* mp = reinterpret_cast<const uint4*>(&S.mass[ms][c0]);  // warp-uniform: broadcast
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 t4 = mp[j];
            pi[4 * j] = t4.x;
            pi[4 * j + 1] = t4.y;
            pi[4 * j + 2] = t4.z;
            pi[4 * j + 3] = t4.w;
          }
        };
        auto load_acc = [&](int c0, uint32_t (&v)[32]) {
          if (c0 + 32 <= N) {
            tmem_ld32(tbase + c0, v);
          } else {  // last chunk of an N = 240 tile: 16 columns (the masses of columns >= N are huge)
            tc::tmem_ld16(tbase + c0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
#pragma unroll
            for (int j = 16; j < 32; ++j) v[j] = 0u;
          }
        };
        // p_i - 2 acc (exact) and the pass test against lim
        auto partial = [&](uint32_t pi, uint32_t v) -> float { return fmaf(-2.0f, __uint_as_float(v), __uint_as_float(pi)); };
        auto passes = [&](uint32_t pi, uint32_t v) -> bool {
          if (FP4) return partial(pi, v) <= limf;
          return static_cast<int32_t>(pi) - 2 * static_cast<int32_t>(v) <= lim;
        };
        auto key_of = [&](uint32_t pi, uint32_t v) -> uint32_t {
          if (FP4) return __float_as_uint(pqf + partial(pi, v) + 8388608.0f) - 0x4B000000u;  // exact int < 2^23
          return static_cast<uint32_t>(pq + static_cast<int32_t>(pi) - 2 * static_cast<int32_t>(v));
        };
        auto release = [&]() {  // this warp's lanes/columns of the accumulator (and the masses) are read
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) {
            tc::mbar_arrive(&S.tempty[acc]);
            tc::mbar_arrive(&S.mempty[ms]);
          }
        };
        if (a.dbg) {
          release();
        } else if (EMIT) {
          // pass 1: which keys pass (one bit per column), then ONE atomic per thread per tile;
          // pass 2 re-reads only the chunks where some lane emits and writes those entries
          uint32_t(*masks)[32] = S.emit_mask[warp - 2];
          int ne = 0;
#pragma unroll 1
          for (int c0 = cb; c0 < ce; c0 += 32) {
            uint32_t v[32], pi[32];
            load_acc(c0, v);
            load_mass(c0, pi);
            tc::tmem_ld_wait();
            uint32_t m4[4] = {0u, 0u, 0u, 0u};  // four independent OR chains
#pragma unroll
            for (int j = 0; j < 32; ++j) m4[j & 3] |= (passes(pi[j], v[j]) ? 1u : 0u) << j;
            uint32_t mk = (m4[0] | m4[1]) | (m4[2] | m4[3]);
            if (ce - c0 < 32) mk &= (1u << (ce - c0)) - 1u;  // columns of the next warp's range
            masks[(c0 - cb) >> 5][lane] = mk;
            ne += __popc(mk);
          }
          int pos = 0;
          if (ne) pos = atomicAdd(a.cnt + q, ne);
          // pass 2: only the columns where some lane emits, one TMEM column (all 32 lanes) per load
#pragma unroll 1
          for (int c0 = cb; c0 < ce; c0 += 32) {
            const uint32_t mk = masks[(c0 - cb) >> 5][lane];
            uint32_t cols = __reduce_or_sync(0xffffffffu, mk);  // warp-uniform
            while (cols) {  // up to 4 columns per TMEM round trip
              int jb[4];
              int nb = 0;
#pragma unroll
              for (int b = 0; b < 4; ++b) {
                jb[b] = cols ? __ffs(cols) - 1 : jb[0];
                if (cols) ++nb;
                cols &= cols - 1;
              }
              uint32_t vb[4];
#pragma unroll
              for (int b = 0; b < 4; ++b)
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                             : "=r"(vb[b])
                             : "r"(tbase + c0 + jb[b])
                             : "memory");
              tc::tmem_ld_wait();
#pragma unroll
              for (int b = 0; b < 4; ++b) {
                const int j = jb[b];
                if (b < nb && ((mk >> j) & 1u)) {
                  if (pos < a.cap) {
                    const int64_t o = static_cast<int64_t>(q) * a.cap + pos;
                    a.buf_id[o] = static_cast<int32_t>(a.id_base + i0 + c0 + j);
                    a.buf_key[o] = key_of(S.mass[ms][c0 + j], vb[b]);
                  }
                  ++pos;
                }
              }
            }
          }
          release();
        } else {
#pragma unroll 1
          for (int c0 = cb; c0 < ce; c0 += 32) {
            uint32_t v[32], pi[32];
            load_acc(c0, v);
            load_mass(c0, pi);
            tc::tmem_ld_wait();
            if (c0 + 32 >= ce) release();
            if (qok) {
              const int64_t ic = i0 + c0;
              KeyT kv[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) kv[j] = static_cast<KeyT>(key_of(pi[j], v[j]));
              KeyT* row = keys + static_cast<int64_t>(q) * a.key_stride + ic;
              const int cols = c0 + 32 <= ce ? 32 : ce - c0;
              if (cols == 32 && ic + 32 <= a.key_stride) {
                uint4* dst = reinterpret_cast<uint4*>(row);
                const uint4* src = reinterpret_cast<const uint4*>(kv);
#pragma unroll
                for (int j = 0; j < static_cast<int>(32 * sizeof(KeyT) / 16); ++j) dst[j] = src[j];
              } else {
                for (int j = 0; j < cols; ++j)
                  if (ic + j < a.n) row[j] = kv[j];
              }
            }
          }
        }
      }
      ++tc_;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, 512);
  }
}

// queries -> [qpad/128][U][128][16 B]: binary -> FP4 nibbles (32 bits per unit), count -> the uint8 counters
__global__ void expand_queries_kernel(int kind, const uint4* __restrict__ SQ /*[nq][cps] row-major chunks*/, int cps,
                                      int nq, int qpad, int U, uint4* __restrict__ Qx) {
  // query-tile-major [qpad/128][U][128][16 B]: a tile's K units are contiguous (one bulk copy per stage)
  const int64_t total = static_cast<int64_t>(U) * qpad;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t qt = t / (static_cast<int64_t>(U) * 128);
    const int rem = static_cast<int>(t - qt * U * 128);
    const int u = rem >> 7, q = static_cast<int>(qt * 128 + (rem & 127));
    uint4 out = make_uint4(0, 0, 0, 0);
    if (q < nq) {
      if (kind == BVSS_SKETCH_BINARY) {
        const uint32_t* row = reinterpret_cast<const uint32_t*>(SQ + static_cast<int64_t>(q) * cps);
        const uint32_t w = row[u];  // sketch bits 32u .. 32u + 31
        out = make_uint4(bits8_to_fp4(w), bits8_to_fp4(w >> 8), bits8_to_fp4(w >> 16), bits8_to_fp4(w >> 24));
      } else {
        out = SQ[static_cast<int64_t>(q) * cps + u];
      }
    }
    Qx[t] = out;
  }
}

// binary database sketches, chunk-major [m/128][n_stride][16 B] -> FP4 operand [m/32][n][16 B]
__global__ void expand_db_fp4_kernel(const uint4* __restrict__ S, int64_t n, int64_t n_stride, int U,
                                     uint4* __restrict__ X) {
  const int64_t total = static_cast<int64_t>(U) * n;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = t % n;
    const int u = static_cast<int>(t / n);
    const uint32_t* ch = reinterpret_cast<const uint32_t*>(S + static_cast<int64_t>(u >> 2) * n_stride + i);
    const uint32_t w = ch[u & 3];
    X[t] = make_uint4(bits8_to_fp4(w), bits8_to_fp4(w >> 8), bits8_to_fp4(w >> 16), bits8_to_fp4(w >> 24));
  }
}

// 16-byte K units per row of the tensor-core operand
int scan_tc_units(int kind, int m) { return kind == BVSS_SKETCH_BINARY ? m / 32 : m / 16; }

int launch_expand_db_fp4(const void* S, int64_t n, int64_t n_stride, int m, void* X, int num_sms, cudaStream_t st) {
  if (n <= 0) return BVSS_OK;
  expand_db_fp4_kernel<<<num_sms * 8, 256, 0, st>>>(static_cast<const uint4*>(S), n, n_stride, m / 32,
                                                    static_cast<uint4*>(X));
  BVSS_TRY(post_launch(__func__, st));
  return BVSS_OK;
}

template <bool FP4, bool EMIT, int MODE, int KS>
static int launch_one(const ScanArgs& a, size_t smem, int grid, cudaStream_t st) {
  auto kfn = scan_tc_kernel<FP4, EMIT, MODE, KS>;
  BVSS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kfn<<<grid, kScanThreads, smem, st>>>(a);
  return BVSS_OK;
}
template <bool FP4, bool EMIT, int MODE>
static int launch_ks(const ScanArgs& a, int ks, size_t smem, int grid, cudaStream_t st) {
  switch (ks) {
    case 8: return launch_one<FP4, EMIT, MODE, 8>(a, smem, grid, st);
    case 7: return launch_one<FP4, EMIT, MODE, 7>(a, smem, grid, st);
    case 6: return launch_one<FP4, EMIT, MODE, 6>(a, smem, grid, st);
    case 5: return launch_one<FP4, EMIT, MODE, 5>(a, smem, grid, st);
    case 4: return launch_one<FP4, EMIT, MODE, 4>(a, smem, grid, st);
    default: return launch_one<FP4, EMIT, MODE, 3>(a, smem, grid, st);
  }
}
template <bool FP4, bool EMIT>
static int launch_mode(const ScanArgs& a, int mode, int ks, size_t smem, int grid, cudaStream_t st) {
  if (mode == MODE_BRES) return launch_ks<FP4, EMIT, MODE_BRES>(a, ks, smem, grid, st);
  if (mode == MODE_ARES) return launch_ks<FP4, EMIT, MODE_ARES>(a, ks, smem, grid, st);
  return launch_ks<FP4, EMIT, MODE_STREAM>(a, ks, smem, grid, st);
}

// Operand residency: the database tile stationary (query tiles streamed from L2) when it fits, else the
// query tile, else both streamed; the stage ring takes the rest of the shared-memory budget.
int scan_tc_mode(int kind, int m) {
  const bool fp4 = kind == BVSS_SKETCH_BINARY;
  const int U = scan_tc_units(kind, m), N = fp4 ? 240 : 256;
  const size_t a_tile = static_cast<size_t>(kScanM) * U * 16, b_tile = static_cast<size_t>(N) * U * 16;
  const size_t a_stage = static_cast<size_t>(kScanM) * kScanStageB, b_stage = static_cast<size_t>(N) * kScanStageB;
  int mode = MODE_STREAM;
  if (b_tile + 4 * a_stage <= static_cast<size_t>(kScanSmemBudget)) mode = MODE_BRES;
  else if (a_tile + 4 * b_stage <= static_cast<size_t>(kScanSmemBudget)) mode = MODE_ARES;
  if (const char* e = getenv("BVSS_SCAN_MODE")) {  // developer switch (0 = query tile resident, 1 = streamed)
    const int want = atoi(e);
    if (want == MODE_STREAM || (want == MODE_ARES && a_tile + 4 * b_stage <= static_cast<size_t>(kScanSmemBudget)))
      mode = want;
  }
  return mode;
}
// Bytes of the database operand one scan launch streams from memory (the algorithmic traffic of K3):
// once per run of a CTA when the database tile is stationary, once per query tile otherwise.
uint64_t scan_tc_db_bytes(int kind, int m, int64_t n, int nq, int num_sms) {
  const int U = scan_tc_units(kind, m), N = kind == BVSS_SKETCH_BINARY ? 240 : 256;
  const int64_t nt = ceil_div<int64_t>(n, N), qt = ceil_div(nq, kScanM);
  const uint64_t row = static_cast<uint64_t>(U) * 16;
  if (scan_tc_mode(kind, m) == MODE_BRES) {
    const int64_t work = nt * qt, grid = work < num_sms ? work : num_sms;
    const int64_t runs = nt + (grid < qt * nt ? grid : 0);  // each database tile once, plus CTA-boundary splits
    return static_cast<uint64_t>(runs < 2 * nt ? runs : 2 * nt) * N * row;
  }
  return static_cast<uint64_t>(qt) * n * row;
}

// keys mode: keys != null; emit mode: tau != null (cnt must be zeroed by the caller).
// S: the DB operand [U][n_stride][16 B]; SQ: query sketches (row-major chunks) expanded into Qx
// ([U][qpad][16 B], qpad >= ceil(nq/128)*128) unless expand == false (Qx already holds them).
int launch_scan_tc(int kind, const void* S, const int32_t* mass, int64_t n, int64_t n_stride, int m, const void* SQ,
                   const int32_t* massQ, int nq, void* Qx, int qpad, void* keys, int64_t key_stride, int* work_counter,
                   int num_sms, cudaStream_t st, const uint32_t* tau, int32_t* cnt, int32_t* buf_id, uint32_t* buf_key,
                   int cap, int64_t id_base, bool expand) {
  (void)work_counter;
  if (nq <= 0 || n <= 0) return BVSS_OK;
  const bool fp4 = kind == BVSS_SKETCH_BINARY;
  const int U = scan_tc_units(kind, m);
  if (U % 8) BVSS_FAIL(BVSS_EUNSUPPORTED, "tensor-core scan needs m %% %d == 0", fp4 ? 256 : 128);
  const int cps = fp4 ? (((m / 32) + 3) / 4) : m / 16;
  if (qpad < ceil_div(nq, kScanM) * kScanM) BVSS_FAIL(BVSS_EINVAL, "scan: query padding %d too small", qpad);
  if (expand) {
    expand_queries_kernel<<<num_sms * 4, 256, 0, st>>>(kind, static_cast<const uint4*>(SQ), cps, nq, qpad, U,
                                                       static_cast<uint4*>(Qx));
    BVSS_TRY(post_launch("expand_queries_kernel", st));
  }
  ScanArgs a;
  a.S = static_cast<const uint4*>(S);
  a.massS = mass;
  a.n = n;
  a.n_stride = n_stride;
  a.Qx = static_cast<const uint4*>(Qx);
  a.massQ = massQ;
  a.nq = nq;
  a.qpad = qpad;
  a.U = U;
  a.keys = keys;
  a.key_stride = key_stride;
  const int N = fp4 ? 240 : 256;
  a.n_tiles = static_cast<int>(ceil_div<int64_t>(n, N));
  a.q_tiles = ceil_div(nq, kScanM);
  a.tau = tau;
  a.cnt = cnt;
  a.buf_id = buf_id;
  a.buf_key = buf_key;
  a.cap = cap;
  a.id_base = id_base;
  a.dbg = getenv("BVSS_SCAN_DBG") ? atoi(getenv("BVSS_SCAN_DBG")) : 0;
  const size_t a_tile = static_cast<size_t>(kScanM) * U * 16, b_tile = static_cast<size_t>(N) * U * 16;
  const size_t a_stage = static_cast<size_t>(kScanM) * kScanStageB, b_stage = static_cast<size_t>(N) * kScanStageB;
  const size_t budget = kScanSmemBudget;
  const int mode = scan_tc_mode(kind, m);
  const size_t fixed = mode == MODE_BRES ? b_tile : (mode == MODE_ARES ? a_tile : 0);
  const size_t stage = (mode == MODE_BRES ? 0 : b_stage) + (mode == MODE_ARES ? 0 : a_stage);
  int ks = static_cast<int>((budget - fixed) / stage);
  if (ks > kScanMaxStages) ks = kScanMaxStages;
  if (ks < 3) BVSS_FAIL(BVSS_EUNSUPPORTED, "scan: stage ring does not fit");
  const size_t smem = fixed + ks * stage + 1024;
  const int64_t work = static_cast<int64_t>(a.n_tiles) * a.q_tiles;
  const int grid = static_cast<int>(work < num_sms ? work : num_sms);
  const bool emit = tau != nullptr;
  if (fp4) {
    if (emit) BVSS_TRY((launch_mode<true, true>(a, mode, ks, smem, grid, st)));
    else BVSS_TRY((launch_mode<true, false>(a, mode, ks, smem, grid, st)));
  } else {
    if (emit) BVSS_TRY((launch_mode<false, true>(a, mode, ks, smem, grid, st)));
    else BVSS_TRY((launch_mode<false, false>(a, mode, ks, smem, grid, st)));
  }
  BVSS_TRY(post_launch(__func__, st));
  return BVSS_OK;
}

}  // namespace bvss
