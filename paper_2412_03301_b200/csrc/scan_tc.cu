// scan_tc.cu — K3 on the 5th-generation tensor cores: the filter scan of Alg 6
// lines 10-13 as an exact unsigned-integer GEMM (tcgen05.mma
// kind::i8, u8 x u8 -> s32 accumulated in TMEM).
//
//   binary : popc(S_Q AND S_i) = sum_j b_Q[j] b_i[j] with every sketch bit expanded
//            to a 0/1 byte; Hamming = p_Q + p_i - 2 popc(AND)          (reading R1)
//   count  : <C_Q, C_i> = sum_j C_Q[j] C_i[j] on the uint8 counters;
//            L2^2 = |C_Q|^2 + |C_i|^2 - 2 <C_Q, C_i>                      (reading R2)
// Both are exact in s32 (max 2048 * 255^2 < 2^31), so the keys are bit-identical
// to the SIMT scan (scan.cu) and to the oracle.
//
// Queries are the STATIONARY operand: A = a tile of 128 query sketches (M = 128,
// one TMEM lane per query), resident in shared memory for a whole work unit when
// 128 x m bytes fit (m <= 1024), else streamed with B.  B = 256 database sets
// (N = 256) streamed through a stage ring in 64-byte K-chunks.  The (query
// tile, database tile) pairs are split into equal contiguous ranges, one per
// persistent CTA (query-tile-major, so a CTA reloads its query tile at most a
// few times).
// Operands use the canonical no-swizzle K-major layout: per 16-byte K unit u a
// [rows][16 B] block (core matrices of 8 rows x 16 B), LBO = rows x 16 B between
// units, SBO = 128 B between 8-row groups.  This is the chunk-major layout the
// sketches are stored in ([m/16][n][16 B], sketch.cu), so count tiles and the
// pre-expanded query tiles arrive by plain contiguous cp.async.bulk copies, and
// binary tiles are expanded bit -> byte by eight expander warps (one database
// set per thread, 128-bit loads prefetched a whole tile ahead in registers).
//
// Because a TMEM lane is a query, the epilogue thread owns one query: its mass
// p_Q and threshold tau_Q live in registers and the per-value work is one IMAD
// and one compare (keys = p_Q + p_i - 2 acc; database masses are warp-uniform
// 128-bit loads).  Emit mode appends (id, key) for key <= tau_Q with one atomic
// per (thread, 32 columns) that emit anything.
//
// CTA = 14 warps: warp 0 bulk copies (query tile; count-mode / streamed-A
// stages), warp 1 TMEM owner + MMA issuer, warps 2-5 epilogue (one per TMEM
// lane quarter, all 256 columns), warps 6-13 bit expansion (binary mode).
// Double-buffered TMEM accumulators (2 x 256 columns).
#include "tc.cuh"

namespace bvss {

constexpr int kScanM = 128;    // queries per tile (MMA M, TMEM lanes)
constexpr int kScanN = 256;    // database sets per tile (MMA N)
constexpr int kScanKB = 64;    // bytes (= u8 elements) of K per stage
constexpr int kScanThreads = 448;  // 14 warps (register file: 128 regs/thread)
constexpr int kScanEpiWarps = 4;
constexpr int kScanExpWarps = 8;
constexpr int kScanResidentMaxM = 1024;  // A resident in smem when 128 x m <= 128 KB
constexpr int kScanRawPer = 8;           // 128-bit raw chunks prefetched per group (expander)

struct ScanArgs {
  int kind;                    // BVSS_SKETCH_BINARY / COUNT_U8
  const uint4* S;              // DB sketches chunk-major: binary [m/128][n][16B bits], count [m/16][n][16B]
  const int32_t* massS;        // [n]
  int64_t n, n_stride;
  const uint4* Qx;             // expanded queries [m/16][qpad][16 B]
  const int32_t* massQ;        // [nq]
  int nq, qpad;
  int m;
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
};

template <int KS>
struct ScanCtl {
  uint64_t full[KS];
  uint64_t empty[KS];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint64_t afull, aempty;
  uint32_t tmem_base;
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
__host__ __device__ __forceinline__ uint32_t idesc_u8_s32(int M, int N) {
  return (2u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
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
// 16 sketch bits -> 16 bytes of 0/1 (bit b of the half -> byte b, little-endian)
__device__ __forceinline__ uint4 expand16(uint32_t half16) {
  uint4 r;
  r.x = ((half16 & 0xFu) * 0x00204081u) & 0x01010101u;
  r.y = (((half16 >> 4) & 0xFu) * 0x00204081u) & 0x01010101u;
  r.z = (((half16 >> 8) & 0xFu) * 0x00204081u) & 0x01010101u;
  r.w = (((half16 >> 12) & 0xFu) * 0x00204081u) & 0x01010101u;
  return r;
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  tc::tmem_ld16(taddr, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
  tc::tmem_ld16(taddr + 16, *reinterpret_cast<uint32_t(*)[16]>(&r[16]));
}

// Work split: the (query tile, database tile) pairs, ordered query-tile-major,
// are cut into gridDim.x equal contiguous ranges, one per CTA (exact balance;
// a CTA changes query tile at most a few times).  A "run" is the part of a
// CTA's range inside one query tile: database tiles [t0, t1) of query tile qt.
struct ScanRun {
  int qt, t0, t1;
};
struct RunIter {
  int64_t f, f1;
  int NT;
  __device__ RunIter(const ScanArgs& a) {
    const int64_t W = static_cast<int64_t>(a.q_tiles) * a.n_tiles;
    f = W * blockIdx.x / gridDim.x;
    f1 = W * (blockIdx.x + 1) / gridDim.x;
    NT = a.n_tiles;
  }
  __device__ bool next(ScanRun& r) {
    if (f >= f1) return false;
    r.qt = static_cast<int>(f / NT);
    r.t0 = static_cast<int>(f - static_cast<int64_t>(r.qt) * NT);
    const int64_t left = f1 - f;
    r.t1 = static_cast<int>(left < NT - r.t0 ? r.t0 + left : NT);
    f += r.t1 - r.t0;
    return true;
  }
};

template <typename KeyT, bool EMIT, bool RESIDENT, int KS>
__global__ void __launch_bounds__(kScanThreads, 1) scan_tc_kernel(ScanArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ ScanCtl<KS> S;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t kBStage = kScanN * kScanKB;                    // 16 KB
  constexpr uint32_t kAStage = RESIDENT ? 0u : kScanM * kScanKB;    // 8 KB streamed A
  constexpr uint32_t kStage = kAStage + kBStage;
  const uint32_t a_res = smem_u32(base);                                                 // resident A
  const uint32_t ring = a_res + (RESIDENT ? static_cast<uint32_t>(kScanM) * a.m : 0u);  // stage ring
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool binary = a.kind == BVSS_SKETCH_BINARY;
  const int KC = a.m / kScanKB;  // stages per tile

  if (tid == 0) {
    const uint32_t fcount = (binary ? kScanExpWarps : 0) + ((!binary || !RESIDENT) ? 1 : 0);
    for (int s = 0; s < KS; ++s) {
      tc::mbar_init(&S.full[s], fcount);
      tc::mbar_init(&S.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&S.tfull[b], 1);
      tc::mbar_init(&S.tempty[b], kScanEpiWarps);
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

  if (warp == 0) {
    // ------------------------------------------------------------ bulk copies
    uint32_t sc = 0, uc = 0;
    const bool per_stage = !binary || !RESIDENT;
    RunIter it(a);
    ScanRun un;
    for (; it.next(un); ++uc) {
      const int q0 = un.qt * kScanM;
      if (RESIDENT) {  // the query tile: m/16 units of [128 rows][16 B]
        tc::mbar_wait(&S.aempty, (uc & 1u) ^ 1u);
        if (lane == 0) arrive_expect_tx(&S.afull, static_cast<uint32_t>(kScanM) * a.m);
        __syncwarp();
        for (int uu = lane; uu < a.m / 16; uu += 32)
          bulk_copy(a_res + uu * (kScanM * 16u), a.Qx + static_cast<int64_t>(uu) * a.qpad + q0, kScanM * 16u,
                    &S.afull);
      }
      if (!per_stage) continue;
      for (int t = un.t0; t < un.t1; ++t) {
        const int64_t i0 = static_cast<int64_t>(t) * kScanN;
        const int rows = static_cast<int>(a.n - i0 < kScanN ? a.n - i0 : kScanN);
        for (int kc = 0; kc < KC; ++kc, ++sc) {
          const int st = sc % KS;
          tc::mbar_wait(&S.empty[st], ((sc / KS) & 1u) ^ 1u);
          const uint32_t sa = ring + st * kStage, sb = sa + kAStage;
          const uint32_t bytes = kAStage + (binary ? 0u : 4u * rows * 16u);
          if (lane == 0) arrive_expect_tx(&S.full[st], bytes);
          __syncwarp();
          if (!RESIDENT && lane < 4) {  // A units 4kc .. 4kc+3
            const int uu = 4 * kc + lane;
            bulk_copy(sa + lane * (kScanM * 16u), a.Qx + static_cast<int64_t>(uu) * a.qpad + q0, kScanM * 16u,
                      &S.full[st]);
          } else if (!binary && lane >= 4 && lane < 8) {  // count-mode DB units
            const int uu = 4 * kc + (lane - 4);
            bulk_copy(sb + (lane - 4) * (kScanN * 16u), a.S + static_cast<int64_t>(uu) * a.n_stride + i0,
                      static_cast<uint32_t>(rows) * 16u, &S.full[st]);
          }
        }
      }
    }
  } else if (warp >= 6) {
    // ------------------------------------------------- bit expansion (binary)
    if (binary) {
      const int r = tid - 192;  // DB row of the tile, 0..255
      const int RC = a.m / 128;  // raw 128-bit chunks per set
      const int G = (RC + kScanRawPer - 1) / kScanRawPer;
      // flat sequence of (run, tile, group) for this CTA; registers hold one group ahead
      RunIter it(a);
      ScanRun un{};
      bool have = it.next(un);
      int t = have ? un.t0 : 0, g = 0;
      uint4 cur[kScanRawPer];
      auto load_group = [&](int tt, int gg, uint4 (&dst)[kScanRawPer]) {
        const int64_t i = static_cast<int64_t>(tt) * kScanN + r;
#pragma unroll
        for (int c = 0; c < kScanRawPer; ++c) {
          const int rc = gg * kScanRawPer + c;
          dst[c] = make_uint4(0, 0, 0, 0);
          if (i < a.n && rc < RC)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(dst[c].x), "=r"(dst[c].y), "=r"(dst[c].z), "=r"(dst[c].w)
                         : "l"(a.S + static_cast<int64_t>(rc) * a.n_stride + i));
        }
      };
      if (have) load_group(t, g, cur);
      uint32_t sc = 0;
      while (have) {
        // next position in the sequence
        int nt = t, ng = g + 1;
        ScanRun nun = un;
        bool nhave = true;
        if (ng == G) {
          ng = 0;
          ++nt;
          if (nt >= nun.t1) {
            nhave = it.next(nun);
            nt = nun.t0;
          }
        }
        uint4 nxt[kScanRawPer];
        if (nhave) load_group(nt, ng, nxt);
#pragma unroll
        for (int c = 0; c < kScanRawPer; ++c) {
          if (g * kScanRawPer + c < RC) {
            const uint32_t w4[4] = {cur[c].x, cur[c].y, cur[c].z, cur[c].w};
#pragma unroll
            for (int h = 0; h < 2; ++h, ++sc) {  // two 64-byte stages per 128-bit chunk
              const int st = sc % KS;
              tc::mbar_wait(&S.empty[st], ((sc / KS) & 1u) ^ 1u);
              const uint32_t sb = ring + st * kStage + kAStage;
#pragma unroll
              for (int uu = 0; uu < 4; ++uu) {
                const int unit = 4 * h + uu;
                const uint4 v = expand16((w4[unit >> 1] >> (16 * (unit & 1))) & 0xFFFFu);
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sb + uu * (kScanN * 16u) + r * 16u),
                             "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                             : "memory");
              }
              tc::fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) tc::mbar_arrive(&S.full[st]);
            }
          }
        }
#pragma unroll
        for (int c = 0; c < kScanRawPer; ++c) cur[c] = nxt[c];
        t = nt;
        g = ng;
        un = nun;
        have = nhave;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = idesc_u8_s32(kScanM, kScanN);
    uint32_t sc = 0, tc_ = 0, uc = 0;
    RunIter it(a);
    ScanRun un;
    for (; it.next(un); ++uc) {
      if (RESIDENT) {
        tc::mbar_wait(&S.afull, uc & 1u);
        tc::fence_after_sync();
      }
      for (int t = un.t0; t < un.t1; ++t, ++tc_) {
        const uint32_t acc = tc_ & 1u;
        tc::mbar_wait(&S.tempty[acc], ((tc_ >> 1) & 1u) ^ 1u);
        tc::fence_after_sync();
        const uint32_t d = tmem + acc * kScanN;
        for (int kc = 0; kc < KC; ++kc, ++sc) {
          const int st = sc % KS;
          tc::mbar_wait(&S.full[st], (sc / KS) & 1u);
          tc::fence_after_sync();
          if (lane == 0) {
            const uint32_t sa = ring + st * kStage, sb = sa + kAStage;
#pragma unroll
            for (int kk = 0; kk < kScanKB / 32; ++kk) {  // K = 32 bytes = 2 units per instruction
              const uint64_t ad = RESIDENT ? kmajor_desc(a_res + (4 * kc + 2 * kk) * (kScanM * 16u), kScanM * 16u, 128u)
                                           : kmajor_desc(sa + 2 * kk * (kScanM * 16u), kScanM * 16u, 128u);
              umma_u8(d, ad, kmajor_desc(sb + 2 * kk * (kScanN * 16u), kScanN * 16u, 128u), idesc,
                      (kc | kk) ? 1u : 0u);
            }
            tc::umma_commit(&S.empty[st]);
            if (kc == KC - 1) tc::umma_commit(&S.tfull[acc]);
          }
          __syncwarp();
        }
      }
      if (RESIDENT) {
        if (lane == 0) tc::umma_commit(&S.aempty);  // the query tile may be replaced
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2-5)
    const int quarter = warp & 3;         // TMEM lane quarter this warp may access
    KeyT* keys = static_cast<KeyT*>(a.keys);
    uint32_t tc_ = 0;
    RunIter it(a);
    ScanRun un;
    while (it.next(un)) {
      const int q = un.qt * kScanM + quarter * 32 + lane;
      const bool qok = q < a.nq;
      const int32_t pq = qok ? __ldg(a.massQ + q) : 0;
      // key <= tau  <=>  p_i - 2 acc <= tau - p_Q   (keys are exact, < 2^31)
      const int32_t lim = EMIT ? (qok ? static_cast<int32_t>(__ldg(a.tau + q)) - pq : -0x40000000) : 0;
      for (int t = un.t0; t < un.t1; ++t, ++tc_) {
        const uint32_t acc = tc_ & 1u;
        const int64_t i0 = static_cast<int64_t>(t) * kScanN;
        tc::mbar_wait(&S.tfull[acc], (tc_ >> 1) & 1u);
        tc::fence_after_sync();
        const uint32_t tbase = tmem + acc * kScanN + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll 1
        for (int c0 = 0; c0 < kScanN; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tbase + c0, v);
          const int64_t ic = i0 + c0;
          int32_t pi[32];
          if (ic + 32 <= a.n) {
            const int4* mp = reinterpret_cast<const int4*>(a.massS + ic);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int4 t4 = __ldg(mp + j);
              pi[4 * j] = t4.x;
              pi[4 * j + 1] = t4.y;
              pi[4 * j + 2] = t4.z;
              pi[4 * j + 3] = t4.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) pi[j] = ic + j < a.n ? __ldg(a.massS + ic + j) : 0x40000000;
          }
          tc::tmem_ld_wait();
          if (c0 + 32 >= kScanN) {  // this warp's lanes of the accumulator are read
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&S.tempty[acc]);
          }
          if (EMIT) {
            uint32_t mask = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              mask |= (pi[j] - 2 * static_cast<int32_t>(v[j]) <= lim ? 1u : 0u) << j;
            if (mask) {  // rare: a few keys per thousand
              const int ne = __popc(mask);
              const int pos0 = atomicAdd(a.cnt + q, ne);
              int e = 0;
#pragma unroll
              for (int j = 0; j < 32; ++j) {  // unrolled: keeps v[] and pi[] in registers
                if ((mask >> j) & 1u) {
                  const int pos = pos0 + e++;
                  if (pos < a.cap) {
                    const int64_t o = static_cast<int64_t>(q) * a.cap + pos;
                    a.buf_id[o] = static_cast<int32_t>(a.id_base + ic + j);
                    a.buf_key[o] = static_cast<uint32_t>(pq + pi[j] - 2 * static_cast<int32_t>(v[j]));
                  }
                }
              }
            }
          } else if (qok) {
            KeyT kv[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) kv[j] = static_cast<KeyT>(pq + pi[j] - 2 * static_cast<int32_t>(v[j]));
            KeyT* row = keys + static_cast<int64_t>(q) * a.key_stride + ic;
            if (ic + 32 <= a.key_stride) {
              uint4* dst = reinterpret_cast<uint4*>(row);
              const uint4* src = reinterpret_cast<const uint4*>(kv);
#pragma unroll
              for (int j = 0; j < static_cast<int>(32 * sizeof(KeyT) / 16); ++j) dst[j] = src[j];
            } else {
              for (int j = 0; j < 32; ++j)
                if (ic + j < a.n) row[j] = kv[j];
            }
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, 512);
  }
}

// queries -> [m/16][qpad][16 B] (binary: bits expanded to 0/1 bytes; count: the uint8 counters)
__global__ void expand_queries_kernel(int kind, const uint4* __restrict__ SQ /*[nq][cps] row-major chunks*/, int cps,
                                      int nq, int qpad, int m, uint4* __restrict__ Qx) {
  const int units = m / 16;
  const int64_t total = static_cast<int64_t>(units) * qpad;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int q = static_cast<int>(t % qpad), u = static_cast<int>(t / qpad);
    uint4 out = make_uint4(0, 0, 0, 0);
    if (q < nq) {
      if (kind == BVSS_SKETCH_BINARY) {
        const uint4 c = SQ[static_cast<int64_t>(q) * cps + (u >> 3)];  // 128-bit chunk holding unit u
        const uint32_t w4[4] = {c.x, c.y, c.z, c.w};
        const int uu = u & 7;
        out = expand16((w4[uu >> 1] >> (16 * (uu & 1))) & 0xFFFFu);
      } else {
        out = SQ[static_cast<int64_t>(q) * cps + u];
      }
    }
    Qx[t] = out;
  }
}

// keys mode: keys != null; emit mode: tau != null (cnt must be zeroed by the caller)
int launch_scan_tc(int kind, const void* S, const int32_t* mass, int64_t n, int64_t n_stride, int m, const void* SQ,
                   const int32_t* massQ, int nq, void* Qx /*workspace [m/16][qpad][16]*/, int qpad, void* keys,
                   int64_t key_stride, int* work_counter, int num_sms, cudaStream_t st, const uint32_t* tau,
                   int32_t* cnt, int32_t* buf_id, uint32_t* buf_key, int cap, int64_t id_base, bool expand) {
  if (nq <= 0 || n <= 0) return BVSS_OK;
  if (m % 128) BVSS_FAIL(BVSS_EUNSUPPORTED, "tensor-core scan needs m %% 128 == 0");
  const int cps = kind == BVSS_SKETCH_BINARY ? (((m / 32) + 3) / 4) : m / 16;
  if (expand) {
    expand_queries_kernel<<<num_sms * 4, 256, 0, st>>>(kind, static_cast<const uint4*>(SQ), cps, nq, qpad, m,
                                                       static_cast<uint4*>(Qx));
    BVSS_TRY(post_launch("expand_queries_kernel", st));
  }
  ScanArgs a;
  a.kind = kind;
  a.S = static_cast<const uint4*>(S);
  a.massS = mass;
  a.n = n;
  a.n_stride = n_stride;
  a.Qx = static_cast<const uint4*>(Qx);
  a.massQ = massQ;
  a.nq = nq;
  a.qpad = qpad;
  a.m = m;
  a.keys = keys;
  a.key_stride = key_stride;
  a.n_tiles = static_cast<int>(ceil_div<int64_t>(n, kScanN));
  a.q_tiles = ceil_div(nq, kScanM);
  if (qpad < a.q_tiles * kScanM) BVSS_FAIL(BVSS_EINVAL, "scan: query padding %d < %d", qpad, a.q_tiles * kScanM);
  a.tau = tau;
  a.cnt = cnt;
  a.buf_id = buf_id;
  a.buf_key = buf_key;
  a.cap = cap;
  a.id_base = id_base;
  (void)work_counter;
  constexpr int KS = 6;
  const bool resident = m <= kScanResidentMaxM;
  const size_t smem = (resident ? static_cast<size_t>(kScanM) * m + static_cast<size_t>(KS) * kScanN * kScanKB
                                : static_cast<size_t>(KS) * (kScanM + kScanN) * kScanKB) + 1024;
  const int64_t work = static_cast<int64_t>(a.n_tiles) * a.q_tiles;
  const int grid = static_cast<int>(work < num_sms ? work : num_sms);
#define BVSS_SCAN_LAUNCH(KT, EM, RES)                                                                     \
  do {                                                                                                    \
    auto kfn = scan_tc_kernel<KT, EM, RES, KS>;                                                           \
    BVSS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem))); \
    cudaFuncAttributes fa;                                                                                \
    BVSS_CUDA(cudaFuncGetAttributes(&fa, kfn));                                                           \
    if (fa.maxThreadsPerBlock < kScanThreads)                                                             \
      BVSS_FAIL(BVSS_ECUDA, "scan_tc_kernel: %d regs/thread, %zu B static smem, %zu B local: max %d threads < %d", \
                fa.numRegs, fa.sharedSizeBytes, fa.localSizeBytes, fa.maxThreadsPerBlock, kScanThreads); \
    kfn<<<grid, kScanThreads, smem, st>>>(a);                                                             \
  } while (0)
#define BVSS_SCAN_LAUNCH2(KT, EM) \
  do {                            \
    if (resident)                 \
      BVSS_SCAN_LAUNCH(KT, EM, true); \
    else                          \
      BVSS_SCAN_LAUNCH(KT, EM, false); \
  } while (0)
  const bool emit = tau != nullptr;
  if (kind == BVSS_SKETCH_BINARY) {
    if (emit) BVSS_SCAN_LAUNCH2(uint16_t, true);
    else BVSS_SCAN_LAUNCH2(uint16_t, false);
  } else {
    if (emit) BVSS_SCAN_LAUNCH2(uint32_t, true);
    else BVSS_SCAN_LAUNCH2(uint32_t, false);
  }
#undef BVSS_SCAN_LAUNCH2
#undef BVSS_SCAN_LAUNCH
  BVSS_TRY(post_launch(__func__, st));
  return BVSS_OK;
}

}  // namespace bvss
