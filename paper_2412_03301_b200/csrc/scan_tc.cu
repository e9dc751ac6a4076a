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
// Tile = 128 database sets (A, M = 128, one TMEM lane each) x 256 queries
// (B, N = 256), K = m in 128-byte chunks; a tcgen05.mma costs ~138 cycles
// whatever N is (tools/microbench_umma.cu), so N = 256 keeps the issue rate at
// the tensor-core peak.  Operands use the canonical no-swizzle K-major layout:
// per 16-byte K unit u a [rows][16 B] block (core matrices of 8 rows x 16 B),
// LBO = rows x 16 B between units, SBO = 128 B between 8-row groups; this is
// exactly the chunk-major layout the sketches are stored in ([m/16][n][16 B],
// sketch.cu), so count tiles and the (pre-expanded) query tiles arrive by plain
// contiguous cp.async.bulk copies, and binary tiles are expanded bit -> byte by
// four producer warps straight into that layout.
//
// CTA = 10 warps: warp 0 bulk copies (query tile; count-mode DB tile), warp 1
// TMEM owner + MMA issuer, warps 2-5 epilogue (keys[q][i] = p_Q + p_i - 2 acc,
// coalesced over sets), warps 6-9 bit expansion (binary mode).  4-stage smem
// ring, double-buffered TMEM accumulators (2 x 256 columns).
#include "tc.cuh"

namespace bvss {

constexpr int kScanM = 128;   // database sets per tile
constexpr int kScanN = 256;   // queries per tile
constexpr int kScanKB = 128;  // bytes (= u8 elements) per K-chunk
constexpr int kScanStages = 4;
constexpr int kScanThreads = 448;  // 0 copies, 1 MMA, 2-5 + 10-13 epilogue, 6-9 bit expansion
constexpr int kScanEpiWarps = 8;

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
  int* work_counter;
  // threshold-emit mode (EMIT = true): keys <= tau[q] are appended to per-query buffers
  const uint32_t* tau;     // [nq]
  int32_t* cnt;            // [nq] entries emitted (may exceed cap: overflow)
  int32_t* buf_id;         // [nq][cap] set ids (+ id_base)
  uint32_t* buf_key;       // [nq][cap] keys
  int cap;
  int64_t id_base;
};

struct ScanCtl {
  uint64_t full[kScanStages];
  uint64_t empty[kScanStages];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  int work[4];  // work ring: (db tile, q tile) pairs claimed by the copy warp
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

template <typename KeyT, bool EMIT>
__global__ void __launch_bounds__(kScanThreads, 1) scan_tc_kernel(ScanArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ ScanCtl S;
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t ring_s = smem_u32(ring);
  constexpr uint32_t kA = kScanM * kScanKB, kB = kScanN * kScanKB, kStage = kA + kB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool binary = a.kind == BVSS_SKETCH_BINARY;
  const int KC = a.m / kScanKB;
  const int total = a.n_tiles * a.q_tiles;

  if (tid == 0) {
    for (int s = 0; s < kScanStages; ++s) {
      tc::mbar_init(&S.full[s], binary ? 1 + 4 : 1);  // copy warp (+ 4 expander warps)
      tc::mbar_init(&S.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&S.tfull[b], 1);
      tc::mbar_init(&S.tempty[b], kScanEpiWarps);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(&S.tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = S.tmem_base;

  // static round-robin over (db tile, q tile), q tile fastest (the db tile stays L2-hot)
  if (warp == 0) {
    // ---------------------------------------------------------- bulk copies
    uint32_t sc = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      const int it = w / a.q_tiles, qt = w % a.q_tiles;
      const int64_t i0 = static_cast<int64_t>(it) * kScanM;
      const int q0 = qt * kScanN;
      const int rows = static_cast<int>(a.n - i0 < kScanM ? a.n - i0 : kScanM);
      for (int kc = 0; kc < KC; ++kc, ++sc) {
        const int st = sc % kScanStages;
        tc::mbar_wait(&S.empty[st], ((sc / kScanStages) & 1u) ^ 1u);
        const uint32_t sa = ring_s + st * kStage, sb = sa + kA;
        const uint32_t bytes = 8u * kScanN * 16u + (binary ? 0u : 8u * rows * 16u);
        if (lane == 0) arrive_expect_tx(&S.full[st], bytes);
        __syncwarp();
        if (lane < 8) {  // query units 8kc .. 8kc+7: [qpad][16 B] blocks of 256 queries
          const int u = 8 * kc + lane;
          bulk_copy(sb + lane * kScanN * 16u, a.Qx + static_cast<int64_t>(u) * a.qpad + q0, kScanN * 16u, &S.full[st]);
        } else if (!binary && lane < 16) {  // count-mode DB units
          const int uu = lane - 8, u = 8 * kc + uu;
          bulk_copy(sa + uu * kScanM * 16u, a.S + static_cast<int64_t>(u) * a.n_stride + i0,
                    static_cast<uint32_t>(rows) * 16u, &S.full[st]);
        }
      }
    }
  } else if (warp >= 6 && warp <= 9) {
    // ------------------------------------------- bit expansion (binary mode)
    if (binary) {
      const int r = tid - 192;  // DB row of the tile, 0..127
      uint32_t sc = 0;
      for (int w = blockIdx.x; w < total; w += gridDim.x) {
        const int it = w / a.q_tiles;
        const int64_t i = static_cast<int64_t>(it) * kScanM + r;
        for (int kc = 0; kc < KC; ++kc, ++sc) {
          const int st = sc % kScanStages;
          uint4 bits = make_uint4(0, 0, 0, 0);
          if (i < a.n) bits = a.S[static_cast<int64_t>(kc) * a.n_stride + i];  // 128 bits of K-chunk kc
          tc::mbar_wait(&S.empty[st], ((sc / kScanStages) & 1u) ^ 1u);
          const uint32_t sa = ring_s + st * kStage;
          const uint32_t w4[4] = {bits.x, bits.y, bits.z, bits.w};
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint4 v = expand16((w4[u >> 1] >> (16 * (u & 1))) & 0xFFFFu);
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sa + u * kScanM * 16u + r * 16u),
                         "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                         : "memory");
          }
          tc::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&S.full[st]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    const uint32_t idesc = idesc_u8_s32(kScanM, kScanN);
    uint32_t sc = 0, tc_ = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x, ++tc_) {
      const uint32_t acc = tc_ & 1u;
      tc::mbar_wait(&S.tempty[acc], ((tc_ >> 1) & 1u) ^ 1u);
      tc::fence_after_sync();
      const uint32_t d = tmem + acc * kScanN;
      for (int kc = 0; kc < KC; ++kc, ++sc) {
        const int st = sc % kScanStages;
        tc::mbar_wait(&S.full[st], (sc / kScanStages) & 1u);
        tc::fence_after_sync();
        if (lane == 0) {
          const uint32_t sa = ring_s + st * kStage, sb = sa + kA;
#pragma unroll
          for (int kk = 0; kk < kScanKB / 32; ++kk) {  // K = 32 bytes = 2 units per instruction
            umma_u8(d, kmajor_desc(sa + 2 * kk * kScanM * 16u, kScanM * 16u, 128u),
                    kmajor_desc(sb + 2 * kk * kScanN * 16u, kScanN * 16u, 128u), idesc, (kc | kk) ? 1u : 0u);
          }
          tc::umma_commit(&S.empty[st]);
          if (kc == KC - 1) tc::umma_commit(&S.tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else {
    // -------------------------------------- epilogue (warps 2-5 and 10-13)
    const int ew = warp & 3;
    const int half = warp >= 10 ? 1 : 0;  // columns [128 half, 128 half + 128)
    const int row = ew * 32 + lane;       // TMEM lane = DB set of the tile
    KeyT* keys = static_cast<KeyT*>(a.keys);
    uint32_t tc_ = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x, ++tc_) {
      const int it = w / a.q_tiles, qt = w % a.q_tiles;
      const int64_t i = static_cast<int64_t>(it) * kScanM + row;
      const int q0 = qt * kScanN + half * (kScanN / 2);
      const bool ok = i < a.n;
      const int32_t pi = ok ? a.massS[i] : 0;
      const uint32_t acc = tc_ & 1u;
      tc::mbar_wait(&S.tfull[acc], (tc_ >> 1) & 1u);
      tc::fence_after_sync();
      const uint32_t tbase = tmem + acc * kScanN + half * (kScanN / 2) + (static_cast<uint32_t>(ew * 32) << 16);
      for (int c0 = 0; c0 < kScanN / 2; c0 += 32) {
        uint32_t v[32];
        tc::tmem_ld16(tbase + c0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
        tc::tmem_ld16(tbase + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
        // query masses (and thresholds) of these 32 columns: warp-uniform loads, overlapped with TMEM
        int32_t pq[32];
        uint32_t tq[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int q = q0 + c0 + j;
          pq[j] = q < a.nq ? __ldg(a.massQ + q) : 0;
          if (EMIT) tq[j] = q < a.nq ? __ldg(a.tau + q) : 0u;
        }
        tc::tmem_ld_wait();
        if (c0 + 32 >= kScanN / 2) {  // this warp's half of the accumulator is read
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&S.tempty[acc]);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int q = q0 + c0 + j;
          const int32_t key = pq[j] + pi - 2 * static_cast<int32_t>(v[j]);
          if (!EMIT) {
            if (q < a.nq && ok) keys[static_cast<int64_t>(q) * a.key_stride + i] = static_cast<KeyT>(key);
          } else {
            const bool pass = ok && q < a.nq && static_cast<uint32_t>(key) <= tq[j];
            const unsigned mask = __ballot_sync(0xffffffffu, pass);
            if (mask) {  // warp-uniform: rare (a few keys per thousand)
              int base = 0;
              if (lane == 0) base = atomicAdd(a.cnt + q, __popc(mask));
              base = __shfl_sync(0xffffffffu, base, 0);
              const int pos = base + __popc(mask & ((1u << lane) - 1u));
              if (pass && pos < a.cap) {
                a.buf_id[static_cast<int64_t>(q) * a.cap + pos] = static_cast<int32_t>(a.id_base + i);
                a.buf_key[static_cast<int64_t>(q) * a.cap + pos] = static_cast<uint32_t>(key);
              }
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
  if (m % kScanKB) BVSS_FAIL(BVSS_EUNSUPPORTED, "tensor-core scan needs m %% 128 == 0");
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
  a.n_tiles = static_cast<int>(ceil_div<int64_t>(n, kScanM));
  a.q_tiles = ceil_div(nq, kScanN);
  a.work_counter = work_counter;
  a.tau = tau;
  a.cnt = cnt;
  a.buf_id = buf_id;
  a.buf_key = buf_key;
  a.cap = cap;
  a.id_base = id_base;
  const size_t smem = static_cast<size_t>(kScanStages) * (kScanM + kScanN) * kScanKB + 1024;
  const int total = a.n_tiles * a.q_tiles;
  const int grid = total < num_sms ? total : num_sms;
#define BVSS_SCAN_LAUNCH(KT, EM)                                                                          \
  do {                                                                                                    \
    auto kfn = scan_tc_kernel<KT, EM>;                                                                    \
    BVSS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem))); \
    kfn<<<grid, kScanThreads, smem, st>>>(a);                                                             \
  } while (0)
  const bool emit = tau != nullptr;
  if (kind == BVSS_SKETCH_BINARY) {
    if (emit) BVSS_SCAN_LAUNCH(uint16_t, true);
    else BVSS_SCAN_LAUNCH(uint16_t, false);
  } else {
    if (emit) BVSS_SCAN_LAUNCH(uint32_t, true);
    else BVSS_SCAN_LAUNCH(uint32_t, false);
  }
#undef BVSS_SCAN_LAUNCH
  BVSS_TRY(post_launch(__func__, st));
  return BVSS_OK;
}

}  // namespace bvss
