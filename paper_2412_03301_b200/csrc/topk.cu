// topk.cu — K6: final top-k with exact fix-up (Alg 6 line 23; Def 5
// P:162-169), and K7: merge of per-shard top-k lists.
//
// K6, one CTA per query: the k-th smallest tensor-core H^2 among the query's
// candidates is found by a 4-round radix select; every candidate whose
// tensor-core H^2 is within 2E of it (E = the rigorous squared-distance error
// bound of the refine arithmetic) is recomputed exactly by fp32
// direct differences sum_k (q_k - v_k)^2 (Def 4 verbatim; one warp per
// candidate, set rows on lanes, query rows in register blocks), and the k
// smallest exact distances are emitted sorted by (distance, id) (reading R4).  The true
// top-k is always inside the window, so the result does not depend on the
// tensor-core rounding.  With E = +inf (refine_terms = 0) the kernel is a plain
// SIMT exact refine of every candidate (correctness anchor).
#include <cstdlib>

#include "tc.cuh"

namespace bvss {

constexpr int kTopkThreads = 256;
constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int kMaxMq = 256;
constexpr int kIB = 16;  // query rows per register block
constexpr int kKB = 32;  // dims per register chunk

struct TopkSmem {
  uint32_t hist[256];
  float rowmin[kTopkWarps][kMaxMq];
  uint32_t wcount;
  uint32_t prefix;
  uint32_t need;
  unsigned long long best;
};

__device__ __forceinline__ float block_max_f(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = red[0];
  for (int i = 1; i < (blockDim.x >> 5); ++i) r = fmaxf(r, red[i]);
  __syncthreads();
  return r;
}

// block-wide sum in a fixed order (butterfly within warps, warps in index order): deterministic
__device__ __forceinline__ float block_sum_f(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = red[0];
  for (int i = 1; i < (blockDim.x >> 5); ++i) r += red[i];
  __syncthreads();
  return r;
}

template <bool VEC>
__device__ __forceinline__ void load_chunk(const float* __restrict__ p, int kb, int d, bool ok, float (&x)[kKB]) {
  if (VEC) {
#pragma unroll
    for (int e = 0; e < kKB; e += 4) {
      float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ok && kb + e < d) t = *reinterpret_cast<const float4*>(p + kb + e);
      x[e] = t.x; x[e + 1] = t.y; x[e + 2] = t.z; x[e + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < kKB; ++e) x[e] = (ok && kb + e < d) ? p[kb + e] : 0.0f;
  }
}

// Exact H^2 of Def 4 by fp32 direct differences, one warp: lane j owns set row
// j (blocks of 32), query rows in register blocks of kIB (uniform, broadcast
// loads), D^2(i,j) = sum_k (q_ik - v_jk)^2 with FMA; min/max on D^2.
template <bool VEC>
__device__ float warp_exact_h2(const float* __restrict__ Q, int mq, const float* __restrict__ Vs, int mi, int d,
                               float* rowmin) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < mq; i += 32) rowmin[i] = __int_as_float(0x7f800000);
  __syncwarp();
  float hv = 0.0f;
  for (int jb = 0; jb < mi; jb += 32) {
    const int j = jb + lane;
    const bool vj = j < mi;
    const float* vrow = Vs + static_cast<int64_t>(vj ? j : 0) * d;
    float colmin = __int_as_float(0x7f800000);
    for (int ib = 0; ib < mq; ib += kIB) {
      float acc[kIB];
#pragma unroll
      for (int ii = 0; ii < kIB; ++ii) acc[ii] = 0.0f;
      for (int kb = 0; kb < d; kb += kKB) {
        float v[kKB];
        load_chunk<VEC>(vrow, kb, d, true, v);
#pragma unroll
        for (int ii = 0; ii < kIB; ++ii) {
          if (ib + ii < mq) {
            float qv[kKB];
            load_chunk<VEC>(Q + static_cast<int64_t>(ib + ii) * d, kb, d, true, qv);
            float s = acc[ii];
#pragma unroll
            for (int e = 0; e < kKB; ++e) {
              const float t = qv[e] - v[e];
              s = __fmaf_rn(t, t, s);
            }
            acc[ii] = s;
          }
        }
      }
#pragma unroll
      for (int ii = 0; ii < kIB; ++ii) {
        if (ib + ii < mq) {
          const float a = vj ? acc[ii] : __int_as_float(0x7f800000);
          colmin = fminf(colmin, a);
          float m = a;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
          if (lane == 0) rowmin[ib + ii] = fminf(rowmin[ib + ii], m);
        }
      }
    }
    hv = fmaxf(hv, vj ? colmin : 0.0f);
  }
  __syncwarp();
  float hq = 0.0f;
  for (int i = lane; i < mq; i += 32) hq = fmaxf(hq, rowmin[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    hv = fmaxf(hv, __shfl_xor_sync(0xffffffffu, hv, o));
    hq = fmaxf(hq, __shfl_xor_sync(0xffffffffu, hq, o));
  }
  return fmaxf(hq, hv);
}

template <bool VEC>
__global__ void __launch_bounds__(kTopkThreads) topk_fixup_kernel(
    const float* __restrict__ approx, const int32_t* __restrict__ cand, const int32_t* __restrict__ count, int T, int k,
    const float* __restrict__ V, const int64_t* __restrict__ off, int64_t id_base, int d, const float* __restrict__ Qv,
    const int64_t* __restrict__ qoff, const float* __restrict__ qnorm, float vmax2, float c1, float c2,
    int exact_all, int64_t* __restrict__ out_ids, float* __restrict__ out_dist, int64_t* __restrict__ fixup_counter) {
  extern __shared__ __align__(16) uint8_t dyn[];
  float* ap = reinterpret_cast<float*>(dyn);                // [T]
  int32_t* win = reinterpret_cast<int32_t*>(ap + T);       // [T]
  float* ex = reinterpret_cast<float*>(win + T);           // [T]
  __shared__ TopkSmem S;
  __shared__ float red[32];
  const int q = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cnt = count ? count[q] : T;
  const int64_t q0 = qoff[q];
  const int mq = static_cast<int>(qoff[q + 1] - q0);
  const int kk = min(k, cnt);
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) ap[i] = approx ? approx[static_cast<int64_t>(q) * T + i] : 0.0f;
  if (threadIdx.x == 0) S.wcount = 0;
  // window threshold W = (k-th smallest tensor-core H^2) + 2E
  float W = __int_as_float(0x7f800000);
  if (!exact_all && kk > 0) {
    float mq2 = 0.0f;
    for (int i = threadIdx.x; i < mq; i += blockDim.x) mq2 = fmaxf(mq2, qnorm[q0 + i]);
    mq2 = block_max_f(mq2, red);
    const float Mq = sqrtf(mq2), Mv = sqrtf(vmax2);
    const float E = c1 * Mq * Mv + c2 * (mq2 + vmax2);
    if (threadIdx.x == 0) {
      S.prefix = 0u;
      S.need = static_cast<uint32_t>(kk);
    }
    for (int rnd = 0; rnd < 4; ++rnd) {  // radix select of the kk-th smallest (uint order of floats >= 0)
      const int shift = 24 - 8 * rnd;
      for (int i = threadIdx.x; i < 256; i += blockDim.x) S.hist[i] = 0u;
      __syncthreads();
      const uint32_t pre = S.prefix;
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        const uint32_t u = __float_as_uint(ap[i]);
        if (rnd == 0 || (u >> (shift + 8)) == pre) atomicAdd(&S.hist[(u >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t need = S.need, run = 0;
        int dsel = 255;
        for (int b = 0; b < 256; ++b) {
          if (run + S.hist[b] >= need) {
            dsel = b;
            break;
          }
          run += S.hist[b];
        }
        S.prefix = (pre << 8) | static_cast<uint32_t>(dsel);
        S.need = need - run;
      }
      __syncthreads();
    }
    W = (__uint_as_float(S.prefix) + 2.0f * E) * (1.0f + 1e-6f);
    if (S.prefix & 0x80000000u) W = __int_as_float(0x7f800000);  // k-th key is a refine sentinel: all in
  }
  __syncthreads();
  for (int i = threadIdx.x; i < cnt; i += blockDim.x)
    if (exact_all || ap[i] <= W) win[atomicAdd(&S.wcount, 1u)] = i;
  __syncthreads();
  const int nw = static_cast<int>(S.wcount);
  // exact recompute of the window: one warp per candidate
  for (int w = warp; w < nw; w += kTopkWarps) {
    const int64_t cid = static_cast<int64_t>(cand[static_cast<int64_t>(q) * T + win[w]]) - id_base;
    const int64_t v0 = off[cid];
    const int mi = static_cast<int>(off[cid + 1] - v0);
    const float h2 = warp_exact_h2<VEC>(Qv + q0 * d, mq, V + v0 * d, mi, d, S.rowmin[warp]);
    if (lane == 0) ex[w] = h2;
  }
  if (threadIdx.x == 0 && fixup_counter) atomicAdd(reinterpret_cast<unsigned long long*>(fixup_counter), nw);
  __syncthreads();
  // k smallest by (exact, id): k rounds of block argmin on a packed 64-bit key
  for (int r = 0; r < k; ++r) {
    unsigned long long best = ~0ull;
    for (int w = threadIdx.x; w < nw; w += blockDim.x) {
      const float e = ex[w];
      if (e < 0.0f) continue;  // taken
      const uint32_t gid = static_cast<uint32_t>(cand[static_cast<int64_t>(q) * T + win[w]]);
      const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(e)) << 32) | gid;
      best = key < best ? key : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
      best = t < best ? t : best;
    }
    if (threadIdx.x == 0) S.best = ~0ull;
    __syncthreads();
    if (lane == 0) atomicMin(&S.best, best);
    __syncthreads();
    const unsigned long long b = S.best;
    if (threadIdx.x == 0) {
      int64_t* oi = out_ids + static_cast<int64_t>(q) * k;
      float* od = out_dist + static_cast<int64_t>(q) * k;
      if (b == ~0ull) {
        oi[r] = -1;
        od[r] = __int_as_float(0x7f800000);
      } else {
        oi[r] = static_cast<int64_t>(static_cast<uint32_t>(b & 0xffffffffull));
        od[r] = sqrtf(__uint_as_float(static_cast<uint32_t>(b >> 32)));
      }
    }
    if (b != ~0ull) {  // mark the winner as taken
      const uint32_t gid = static_cast<uint32_t>(b & 0xffffffffull);
      for (int w = threadIdx.x; w < nw; w += blockDim.x)
        if (static_cast<uint32_t>(cand[static_cast<int64_t>(q) * T + win[w]]) == gid) ex[w] = -1.0f;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K6 v2: the same window rule, with the exact recompute run by the whole CTA on
// shared-memory tiles.  Per query (one CTA, 256 threads):
//   1. radix select of the k-th smallest tensor-core H^2 (4 x 8-bit rounds,
//      smem histogram, warp-parallel digit search) and the window
//      W = H^2_(k) + 2E; the window's candidate slots go to global scratch;
//   2. for every window candidate, Def 4 by fp32 direct differences: the query
//      rows (resident, blocks of RB rows) and the candidate's rows (RB-row
//      blocks, cp.async staging; two CTAs per SM overlap staging and math) are
//      tiles in smem; each thread
//      owns 2 x 2 (query row, set row) pairs over a slice of the d dimensions
//      (the slices cover d as evenly as the pair count allows), partial sums
//      meet in smem, and the row / column minima of D^2 are kept with
//      shared-memory atomicMin on the (non-negative) float bits;
//   3. the k smallest exact distances by (distance, id).
constexpr int kTxThreads = 256;

constexpr int kTxCache = 256;  // window candidates whose row ranges are cached in smem

struct TxSmem {
  int64_t jv0[kTxCache];  // first row and row count of window candidate w
  int jmi[kTxCache];
  uint32_t hist[256];
  uint32_t rowmin[256];   // min_v D^2 of each query row (kMaxMq)
  uint32_t colmin[32];    // min_q D^2 of each set row of the current block
  uint32_t prefix, need, wcount;
  int nb, rows;           // SMALL: candidates and set rows of the current batch
  float hv;
  unsigned long long best;
};

__device__ __forceinline__ void stage_rows(float* dst, int stride4, const float* __restrict__ src, int rows, int d,
                                           int d4) {
  // rows x d fp32 -> smem rows of stride4 float4 (zero-padded to d4 float4); 16-byte cp.async when d % 4 == 0
  if ((d & 3) == 0) {
    const int total = rows * d4;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int r = t / d4, c = t - r * d4;
      tc::cp_async16(smem_u32(dst + (static_cast<int64_t>(r) * stride4 + c) * 4), src + static_cast<int64_t>(r) * d + 4 * c, 16);
    }
  } else {
    const int total = rows * d4 * 4;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int r = t / (d4 * 4), c = t - r * (d4 * 4);
      dst[static_cast<int64_t>(r) * stride4 * 4 + c] = c < d ? src[static_cast<int64_t>(r) * d + c] : 0.0f;
    }
  }
  tc::cp_async_commit();
}

// SMALL (host-chosen: every set and query set has <= 32 rows, d % 4 == 0): phase 2 packs the set rows of
// the window candidates densely onto warp lanes (see the comment at the SMALL branch)
__device__ int g_k6prof_on;                // debug (BVSS_K6_PROF): per-phase clock sums of the SMALL kernel
__device__ unsigned long long g_k6prof[8];

constexpr int kSmRows = 1024;  // SMALL: set rows per batch (their column minima live in smem)
constexpr int kSmRm = 1024;    // SMALL: (candidate, query row) row minima per batch
__host__ __device__ constexpr int nch_pad(int d4) { return (d4 + 7) & ~7; }  // SMALL: d4 in whole 8-float4 chunks

// SMALL phase 2, one full chunk (8 float4 of d) of a 64-row block: lane rows `lane` and `lane + 32` of the
// ring slot (row stride 9 float4) against this warp's GN query rows; qc = the transposed query tile at
// (first dim of the chunk, first query row of the warp): column-major [d4][32] float4, so the GN rows of a
// dim sit at immediate offsets (broadcast reads).  a0 / a1: D^2 partial sums (even / odd dims in .x / .y).
template <int GN>
__device__ __forceinline__ void k6_chunk(const float4* __restrict__ slot, int lane, const float4* __restrict__ qc,
                                         float2 (&a0)[8], float2 (&a1)[8]) {
  const float2 m1 = make_float2(-1.0f, -1.0f);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float4 va = slot[lane * 9 + c], vb = slot[(lane + 32) * 9 + c];
    const float2 va0 = make_float2(va.x, va.y), va1 = make_float2(va.z, va.w);
    const float2 vb0 = make_float2(vb.x, vb.y), vb1 = make_float2(vb.z, vb.w);
#pragma unroll
    for (int i = 0; i < GN; ++i) {
      const float4 q = qc[c * 32 + i];
      const float2 q0 = make_float2(q.x, q.y), q1 = make_float2(q.z, q.w);
      const float2 ta0 = __ffma2_rn(va0, m1, q0), ta1 = __ffma2_rn(va1, m1, q1);
      const float2 tb0 = __ffma2_rn(vb0, m1, q0), tb1 = __ffma2_rn(vb1, m1, q1);
      a0[i] = __ffma2_rn(ta0, ta0, a0[i]);
      a1[i] = __ffma2_rn(tb0, tb0, a1[i]);
      a0[i] = __ffma2_rn(ta1, ta1, a0[i]);
      a1[i] = __ffma2_rn(tb1, tb1, a1[i]);
    }
  }
}

template <bool SMALL>
__global__ void __launch_bounds__(kTxThreads, 2) topk_exact_kernel(
    const float* __restrict__ approx, const int32_t* __restrict__ cand, const int32_t* __restrict__ count, int T, int k,
    const float* __restrict__ V, const int64_t* __restrict__ off, int64_t id_base, int d, int d4, int stride4, int RB, int RBV,
    const float* __restrict__ Qv, const int64_t* __restrict__ qoff, const float* __restrict__ qnorm, float vmax2,
    float c1, float c2, int exact_all, int32_t* __restrict__ win_g, float* __restrict__ ex_g,
    int64_t* __restrict__ out_ids, float* __restrict__ out_dist, int64_t* __restrict__ fixup_counter, int metric,
    const float* __restrict__ approx_err) {
  extern __shared__ __align__(16) float txs[];
  float* Qs = txs;                                            // [RB][stride4*4] query rows
  float* Vs0 = Qs + static_cast<int64_t>(RB) * stride4 * 4;     // [2][RBV][stride4*4] set rows, double-buffered:
  float* red = Vs0 + static_cast<int64_t>(2 * RBV) * stride4 * 4;  // the next block stages during this one's math
  __shared__ TxSmem S;
  __shared__ float bred[32];
  const int q = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cnt = count ? count[q] : T;
  const int64_t q0 = qoff[q];
  const int mq = static_cast<int>(qoff[q + 1] - q0);
  const int kk = min(k, cnt);
  const float* ap = approx ? approx + static_cast<int64_t>(q) * T : nullptr;
  // MeanMin with per-candidate error bounds e: select on the upper bounds a + e, test the lower bounds a - e
  const float* aerr = (metric == 1 && approx_err) ? approx_err + static_cast<int64_t>(q) * T : nullptr;
  const int32_t* cq = cand + static_cast<int64_t>(q) * T;
  int32_t* win = win_g + static_cast<int64_t>(q) * T;
  float* ex = ex_g + static_cast<int64_t>(q) * T;
  if (tid == 0) S.wcount = 0;
  const bool prof = SMALL && g_k6prof_on;
  if (SMALL) {  // stage the transposed query tile QT[c][r] (row r, float4 c; zero past d) under phase 1
    const int d4p = nch_pad(d4);
    float4* QT = reinterpret_cast<float4*>(Qs);
    for (int t = tid; t < mq * d4p; t += blockDim.x) {
      const int r = t / d4p, c = t - r * d4p;
      tc::cp_async16(smem_u32(QT + c * 32 + r), Qv + (q0 + r) * d + 4 * (c < d4 ? c : 0), c < d4 ? 16u : 0u);
    }
    tc::cp_async_commit();
  }
  long long pt0 = prof ? clock64() : 0, pt1 = 0, pt2 = 0, pt3 = 0;
  // ---- 1. window
  float W = __int_as_float(0x7f800000);
  if (!exact_all && kk > 0) {
    float mq2 = 0.0f;
    for (int i = tid; i < mq; i += blockDim.x) mq2 = fmaxf(mq2, qnorm[q0 + i]);
    mq2 = block_max_f(mq2, bred);
    const float E = c1 * sqrtf(mq2) * sqrtf(vmax2) + c2 * (mq2 + vmax2);
    uint32_t pre = 0u, need = static_cast<uint32_t>(kk);
    constexpr int kReg = 8;  // candidates held in registers per thread (cnt <= 2048); beyond: re-read
    uint32_t ur[kReg];
#pragma unroll
    for (int e = 0; e < kReg; ++e) {
      const int i = tid + e * kTxThreads;
      ur[e] = i < cnt ? __float_as_uint(aerr ? ap[i] + aerr[i] : ap[i]) : 0xFFFFFFFFu;
    }
    for (int rnd = 0; rnd < 4; ++rnd) {  // radix select of the kk-th smallest (uint order of floats >= 0)
      const int shift = 24 - 8 * rnd;
      S.hist[tid] = 0u;
      __syncthreads();
#pragma unroll
      for (int e = 0; e < kReg; ++e) {  // warp-aggregated: the values cluster in a few bins
        const uint32_t u = ur[e];
        const bool in = tid + e * kTxThreads < cnt && (rnd == 0 || (u >> (shift + 8)) == pre);
        const uint32_t bin = in ? ((u >> shift) & 255u) : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, bin);
        if (in && lane == __ffs(peers) - 1) atomicAdd(&S.hist[bin], static_cast<uint32_t>(__popc(peers)));
      }
      for (int i = tid + kReg * kTxThreads; i < cnt; i += blockDim.x) {
        const uint32_t u = __float_as_uint(aerr ? ap[i] + aerr[i] : ap[i]);
        if (rnd == 0 || (u >> (shift + 8)) == pre) atomicAdd(&S.hist[(u >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (warp == 0) {  // lane l owns bins 8l .. 8l+7
        uint32_t h[8], sum = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          h[b] = S.hist[8 * lane + b];
          sum += h[b];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const uint32_t excl = incl - sum;
        const unsigned hit = __ballot_sync(0xffffffffu, incl >= need && excl < need);
        const int owner = __ffs(hit) - 1;
        if (lane == owner) {
          uint32_t run = excl;
          int dsel = 8 * lane + 7;
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            if (run + h[b] >= need) {
              dsel = 8 * lane + b;
              break;
            }
            run += h[b];
          }
          S.prefix = (pre << 8) | static_cast<uint32_t>(dsel);
          S.need = need - run;
        }
      }
      __syncthreads();
      pre = S.prefix;
      need = S.need;
    }
    // Hausdorff / Min: values are squared distances, each within E of the exact one; MeanMin: values are
    // distances (the mean of sqrt(min_v D^2)), each row term within sqrt(E) since |sqrt a - sqrt b| <=
    // sqrt|a - b|, and the fp32 sums add a few ulps per term (the 2e-5 slack)
    W = aerr ? __uint_as_float(pre) * (1.0f + 2e-5f) + 1e-30f  // the k-th smallest upper bound
        : metric == 1 ? (__uint_as_float(pre) + 2.0f * sqrtf(E)) * (1.0f + 2e-5f) + 1e-30f
                      : (__uint_as_float(pre) + 2.0f * E) * (1.0f + 1e-6f);
    // the k-th smallest key is a refine sentinel (< 0: a candidate the tensor path did not take): fewer than
    // k candidates have a tensor-core value, so every candidate is in the window
    if (pre & 0x80000000u) W = __int_as_float(0x7f800000);
  }
  __syncthreads();
  if (exact_all) {
    for (int i = tid; i < cnt; i += blockDim.x) win[i] = i;
    if (tid == 0) S.wcount = cnt;
  } else {
    for (int i = tid; i < cnt; i += blockDim.x)
      if ((aerr ? ap[i] - aerr[i] : ap[i]) <= W) win[atomicAdd(&S.wcount, 1u)] = i;
  }
  __syncthreads();
  const int nw = static_cast<int>(S.wcount);
  if (tid == 0 && fixup_counter) atomicAdd(reinterpret_cast<unsigned long long*>(fixup_counter), nw);
  // ---- 2. exact H^2 of every window candidate
  if (prof) pt1 = clock64();
  if constexpr (SMALL) {
    // Set rows on lanes, packed, staged through shared memory.  The window candidates' rows are concatenated
    // (candidate order) into blocks of kRB = 64 rows; lane l of a warp owns rows l and l + 32 of a block, so
    // a short set never leaves a lane idle (sizes 4..32 left ~45 % of the lanes of a one-candidate-per-warp
    // mapping empty).  The CTA is two warp groups of four warps; a group walks its blocks (wg, wg + 2, ...)
    // in d-chunks of kCH float4: the group's 128 threads copy a chunk of all 64 rows with coalesced 16-byte
    // cp.async (8 threads per 128-byte row piece) into a two-slot ring, the next chunk loading during this
    // one's math, and each of the four warps takes a quarter of the query rows (<= 8, acc in registers).
    // Staging matters: per-lane global loads of 32 different rows cost 32 L1 wavefronts per instruction and
    // saturated the LSU data pipe (83 %); here a warp's copy instruction covers 4 rows (4 wavefronts).
    // acc = D^2(q_i, v) by fp32 direct differences (FFMA2); the query rows are broadcast smem reads, each
    // feeding 8 FFMA2 (two set rows).  Row minima: a segmented min over the lanes of one candidate
    // (shuffles), then one smem atomicMin per (candidate, query row) by the segment's first lane; column
    // minima: smem atomicMin per (row, warp).  Batches bound the smem minima (kSmRows rows, kSmRm minima).
    constexpr int kRB = 64, kCH = 8, kRS = kCH + 1, kD = 2;
    const int d4p = nch_pad(d4);                                                    // d4 rounded up to kCH
    float4* QT = reinterpret_cast<float4*>(Qs);                                      // [d4p][32] transposed
    float4* ring = QT + static_cast<int64_t>(d4p) * 32;                              // [2][kD][kRB][kRS]
    int* rs = reinterpret_cast<int*>(ring + 2 * kD * kRB * kRS);                              // [kTxCache + 1]
    uint32_t* rowm = reinterpret_cast<uint32_t*>(rs + kTxCache + 1);                         // [kSmRm]
    uint32_t* colm = rowm + kSmRm;                                                           // [kSmRows]
    uint8_t* rc = reinterpret_cast<uint8_t*>(colm + kSmRows);                                // row -> candidate
    // (the transposed query tile was staged at kernel start, overlapping phase 1)
    const int wg = warp >> 2, w4 = warp & 3, tg = tid & 127;
    // this warp's query rows: a quarter of them (<= 8) on the group's own blocks; an eighth on a shared last
    // block (odd block count: both groups take it, each half of the query rows, so neither idles)
    const int i0q = w4 * mq / 4, gnq = (w4 + 1) * mq / 4 - i0q;
    const int i0e = (wg * 4 + w4) * mq / 8, gne = (wg * 4 + w4 + 1) * mq / 8 - i0e;
    const int nch = (d4 + kCH - 1) / kCH;
    const int crow = tg >> 3, ccol = tg & 7;  // copy role: rows crow + 16 j (j < 4), float4 column ccol
    for (int xb = 0; xb < nw;) {
      const int nc = min(kTxCache, nw - xb);
      for (int t = tid; t < nc; t += blockDim.x) {
        const int64_t cid = static_cast<int64_t>(cq[win[xb + t]]) - id_base;
        const int64_t v0 = off[cid];
        S.jv0[t] = v0;
        S.jmi[t] = static_cast<int>(off[cid + 1] - v0);
      }
      __syncthreads();
      if (warp == 0) {  // the batch: the longest prefix within both smem caps (a single candidate always fits)
        int run = 0, nb = 0;
        for (int t0 = 0; t0 < nc; t0 += 32) {
          const int t = t0 + lane;
          const int mi = t < nc ? S.jmi[t] : 0;
          int incl = mi;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
          }
          const int end = run + incl;
          const bool fits = t < nc && end <= kSmRows && (t + 1) * mq <= kSmRm;
          const int nf = __popc(__ballot_sync(0xffffffffu, fits));  // fits is a prefix of the lanes
          if (lane < nf) rs[t] = end - mi;
          nb = t0 + nf;
          if (nf > 0) run = __shfl_sync(0xffffffffu, end, nf - 1);
          if (nf < 32) break;
        }
        if (lane == 0) {
          rs[nb] = run;
          S.nb = nb;
          S.rows = run;
        }
      }
      __syncthreads();
      const int nb = S.nb, rows = S.rows;
      for (int t = tid; t < nb; t += blockDim.x)
        for (int r = rs[t]; r < rs[t + 1]; ++r) rc[r] = static_cast<uint8_t>(t);
      for (int t = tid; t < nb * mq; t += blockDim.x) rowm[t] = 0x7f800000u;
      for (int t = tid; t < rows; t += blockDim.x) colm[t] = 0x7f800000u;
      tc::cp_async_wait<0>();
      __syncthreads();
      if (prof && xb == 0) pt2 = clock64();
      const long long pj0 = prof ? clock64() : 0;
      const int nrb = (rows + kRB - 1) / kRB;
      const int npair = nrb >> 1;                      // blocks 2b + wg (b < npair) are the group's own
      const int nel = (npair + (nrb & 1)) * nch;       // (block, chunk) elements of this group
      auto blk = [&](int bi) { return bi < npair ? 2 * bi + wg : nrb - 1; };
      const float4* src[4];
      auto issue = [&](int e) {  // cp.async of element e into ring slot e % kD (one commit group per call)
        if (e < nel) {
          const int bi = e / nch, ch = e - bi * nch;
          if (ch == 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int rr = min(blk(bi) * kRB + crow + 16 * j, rows - 1);  // past the end: a copy of the last row
              const int xx = rc[rr];
              src[j] = reinterpret_cast<const float4*>(V + (S.jv0[xx] + (rr - rs[xx])) * d);
            }
          }
          float4* dst = ring + static_cast<int64_t>((wg * kD + (e & 1)) * kRB) * kRS;
          const int c = ch * kCH + ccol;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            tc::cp_async16(smem_u32(dst + (crow + 16 * j) * kRS + ccol), src[j] + (c < d4 ? c : 0), c < d4 ? 16u : 0u);
        }
        tc::cp_async_commit();
      };
      float2 a0[8], a1[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a0[i] = a1[i] = make_float2(0.f, 0.f);
      issue(0);
      for (int e = 0; e < nel; ++e) {
        tc::cp_async_wait<0>();
        if (wg == 0)  // element e landed; e - 1 consumed by the whole group
          asm volatile("bar.sync 1, 128;" ::: "memory");
        else
          asm volatile("bar.sync 2, 128;" ::: "memory");
        issue(e + 1);
        const int bi = e / nch, ch = e - bi * nch;
        const bool shared_blk = bi >= npair;
        const int i0 = shared_blk ? i0e : i0q, gn = shared_blk ? gne : gnq;
        const float4* slot = ring + static_cast<int64_t>((wg * kD + (e & 1)) * kRB) * kRS;
        const float4* qc = QT + static_cast<int64_t>(ch * kCH) * 32 + i0;  // past d: zero query and set dims
        switch (gn) {  // warp-uniform: branch-free unrolled math
          case 1: k6_chunk<1>(slot, lane, qc, a0, a1); break;
          case 2: k6_chunk<2>(slot, lane, qc, a0, a1); break;
          case 3: k6_chunk<3>(slot, lane, qc, a0, a1); break;
          case 4: k6_chunk<4>(slot, lane, qc, a0, a1); break;
          case 5: k6_chunk<5>(slot, lane, qc, a0, a1); break;
          case 6: k6_chunk<6>(slot, lane, qc, a0, a1); break;
          case 7: k6_chunk<7>(slot, lane, qc, a0, a1); break;
          case 8: k6_chunk<8>(slot, lane, qc, a0, a1); break;
          default: break;
        }
        if (ch == nch - 1) {  // block done: row / column minima of its two 32-row halves
          auto fold = [&](float2(&a)[8], int r) {
            const bool valid = r < rows;
            const int x = rc[valid ? r : rows - 1];
            const int key = valid ? x : -1 - lane;  // idle lanes: unique keys
            unsigned same = 0u;
#pragma unroll
            for (int b = 0; b < 5; ++b) {
              const int ko = __shfl_down_sync(0xffffffffu, key, 1 << b);
              if (lane + (1 << b) < 32 && ko == key) same |= 1u << b;
            }
            const int kprev = __shfl_up_sync(0xffffffffu, key, 1);
            const bool head = valid && (lane == 0 || kprev != key);
            float cm = __int_as_float(0x7f800000);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (i >= gn) break;
              float m = a[i].x + a[i].y;
              a[i] = make_float2(0.f, 0.f);
              cm = fminf(cm, m);
#pragma unroll
              for (int b = 0; b < 5; ++b) {
                const float u = __shfl_down_sync(0xffffffffu, m, 1 << b);
                if (same & (1u << b)) m = fminf(m, u);
              }
              if (head) atomicMin(&rowm[x * mq + i0 + i], __float_as_uint(m));
            }
            if (valid && gn > 0) atomicMin(&colm[r], __float_as_uint(cm));
          };
          const int rbase = blk(bi) * kRB;
          fold(a0, rbase + lane);
          fold(a1, rbase + 32 + lane);
        }
      }
      tc::cp_async_wait<0>();
      if (prof && lane == 0) atomicAdd(&g_k6prof[6], static_cast<unsigned long long>(clock64() - pj0));
      __syncthreads();
      for (int t = warp; t < nb; t += kTxThreads / 32) {  // H^2 = max(max_q min_v D^2, max_v min_q D^2) etc.
        const int mi = rs[t + 1] - rs[t];
        const float rm = lane < mq ? __uint_as_float(rowm[t * mq + lane]) : 0.0f;
        float val;
        if (metric == 1) {
          float sq = lane < mq ? sqrtf(rm) : 0.0f;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
          val = sq / static_cast<float>(mq);  // MeanMin (a distance)
        } else if (metric == 2) {
          val = __uint_as_float(__reduce_min_sync(0xffffffffu, lane < mq ? __float_as_uint(rm) : 0x7f800000u));
        } else {
          const uint32_t hq = __reduce_max_sync(0xffffffffu, __float_as_uint(rm));
          const uint32_t hv = __reduce_max_sync(0xffffffffu, lane < mi ? colm[rs[t] + lane] : 0u);
          val = __uint_as_float(max(hq, hv));
        }
        if (lane == 0) ex[xb + t] = val;
      }
      __syncthreads();
      xb += nb;
    }
  } else {
  const int nqb = (mq + RB - 1) / RB;
  const int rowsq0 = min(RB, mq);
  if (nqb == 1) stage_rows(Qs, stride4, Qv + q0 * d, rowsq0, d, d4);
  for (int i = tid; i < mq; i += blockDim.x) S.rowmin[i] = 0x7f800000u;
  if (tid < 32) S.colmin[tid] = 0x7f800000u;
  if (tid == 0) S.hv = 0.0f;
  // the window candidates' row ranges, gathered in parallel once (smem for the first kTxCache entries)
  for (int x = tid; x < min(nw, kTxCache); x += blockDim.x) {
    const int64_t cid = static_cast<int64_t>(cq[win[x]]) - id_base;
    const int64_t v0 = off[cid];
    S.jv0[x] = v0;
    S.jmi[x] = static_cast<int>(off[cid + 1] - v0);
  }
  __syncthreads();
  {
  // job sequence: (window entry w, set-row block vb)
  auto job_rows = [&](int w, int vb, const float** src, int* rows) {
    int64_t v0;
    int mi;
    if (w < kTxCache) {
      v0 = S.jv0[w];
      mi = S.jmi[w];
    } else {
      const int64_t cid = static_cast<int64_t>(cq[win[w]]) - id_base;
      v0 = off[cid];
      mi = static_cast<int>(off[cid + 1] - v0);
    }
    *src = V + (v0 + static_cast<int64_t>(vb) * RBV) * d;
    *rows = min(RBV, mi - vb * RBV);
    return mi;
  };
  int w = 0, vb = 0, buf = 0;
  if (nw > 0) {  // stage the first job
    const float* src0;
    int rows0;
    job_rows(0, 0, &src0, &rows0);
    stage_rows(Vs0, stride4, src0, rows0, d, d4);
  }
  while (w < nw) {
    const float* src;
    int rowsv;
    const int mi = job_rows(w, vb, &src, &rowsv);
    int nw_ = w, nvb = vb + 1;  // next job
    if (nvb * RBV >= mi) {
      nw_ = w + 1;
      nvb = 0;
    }
    if (nw_ < nw) {  // prefetch the next job into the other buffer, then wait for this one (all but 1 group)
      const float* nsrc;
      int nrows;
      job_rows(nw_, nvb, &nsrc, &nrows);
      stage_rows(Vs0 + static_cast<int64_t>(buf ^ 1) * RBV * stride4 * 4, stride4, nsrc, nrows, d, d4);
      tc::cp_async_wait<1>();
    } else {
      tc::cp_async_wait<0>();
    }
    __syncthreads();
    const float* Vb = Vs0 + static_cast<int64_t>(buf) * RBV * stride4 * 4;
    for (int qb = 0; qb < nqb; ++qb) {
      const int rowsq = min(RB, mq - qb * RB);
      if (nqb > 1) {  // query blocks restaged per (candidate block, query block): only for m_q > RB
        __syncthreads();
        stage_rows(Qs, stride4, Qv + (q0 + static_cast<int64_t>(qb) * RB) * d, rowsq, d, d4);
        tc::cp_async_wait<0>();
        __syncthreads();
      }
      const int ti_n = (rowsq + 1) >> 1, tj_n = (rowsv + 1) >> 1;
      const int ntile = ti_n * tj_n;
      const int dsplit = max(1, min(kTxThreads / ntile, d4));
      const int tile = tid % ntile, split = tid / ntile;
      // packed fp32x2 math (sm_100 FFMA2: half the instructions of scalar FP32): each accumulator holds
      // the even- and odd-dimension partial sums of one (query row, set row) pair, folded at the end
      float2 acc2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      // thread (tile, split): query rows {it, it + ti_n}, set rows {jt, jt + tj_n} (consecutive lanes take
      // consecutive set rows: conflict-free 16-byte reads at the odd row stride), dims of slice `split`
      if (split < dsplit) {
        const int i0 = tile / tj_n, j0 = tile % tj_n;
        const int i1 = min(i0 + ti_n, rowsq - 1), j1 = min(j0 + tj_n, rowsv - 1);
        const float4* qa = reinterpret_cast<const float4*>(Qs) + i0 * stride4;
        const float4* qb4 = reinterpret_cast<const float4*>(Qs) + i1 * stride4;
        const float4* va = reinterpret_cast<const float4*>(Vb) + j0 * stride4;
        const float4* vb4 = reinterpret_cast<const float4*>(Vb) + j1 * stride4;
        const int kb = split * d4 / dsplit, ke = (split + 1) * d4 / dsplit;
        const float2 m1 = make_float2(-1.0f, -1.0f);
#pragma unroll 4
        for (int c = kb; c < ke; ++c) {
          const float4 x0 = qa[c], x1 = qb4[c], y0 = va[c], y1 = vb4[c];
          const float2 x0a = make_float2(x0.x, x0.y), x0b = make_float2(x0.z, x0.w);
          const float2 x1a = make_float2(x1.x, x1.y), x1b = make_float2(x1.z, x1.w);
          const float2 y0a = make_float2(y0.x, y0.y), y0b = make_float2(y0.z, y0.w);
          const float2 y1a = make_float2(y1.x, y1.y), y1b = make_float2(y1.z, y1.w);
          // t = x - y exactly rounded (fma(-1, y, x)), then acc += t * t
#define BVSS_DD2(A, X, Y)                     \
  {                                           \
    const float2 t_ = __ffma2_rn(Y, m1, X);   \
    A = __ffma2_rn(t_, t_, A);                \
  }
          BVSS_DD2(acc2[0], x0a, y0a)
          BVSS_DD2(acc2[0], x0b, y0b)
          BVSS_DD2(acc2[1], x0a, y1a)
          BVSS_DD2(acc2[1], x0b, y1b)
          BVSS_DD2(acc2[2], x1a, y0a)
          BVSS_DD2(acc2[2], x1b, y0b)
          BVSS_DD2(acc2[3], x1a, y1a)
          BVSS_DD2(acc2[3], x1b, y1b)
#undef BVSS_DD2
        }
      }
      float acc[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = acc2[i].x + acc2[i].y;
      if (dsplit > 1) {
        reinterpret_cast<float4*>(red)[tid] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        __syncthreads();
        if (tid < ntile) {
          for (int sp = 1; sp < dsplit; ++sp) {
            const float4 r = reinterpret_cast<const float4*>(red)[sp * ntile + tid];
            acc[0] += r.x;
            acc[1] += r.y;
            acc[2] += r.z;
            acc[3] += r.w;
          }
        }
      }
      if (tid < ntile) {
        const int i0 = tid / tj_n, j0 = tid % tj_n;
        const bool iv1 = i0 + ti_n < rowsq, jv1 = j0 + tj_n < rowsv;
        const float r0 = fminf(acc[0], jv1 ? acc[1] : acc[0]);
        atomicMin(&S.rowmin[qb * RB + i0], __float_as_uint(r0));
        if (iv1) atomicMin(&S.rowmin[qb * RB + i0 + ti_n], __float_as_uint(fminf(acc[2], jv1 ? acc[3] : acc[2])));
        atomicMin(&S.colmin[j0], __float_as_uint(fminf(acc[0], iv1 ? acc[2] : acc[0])));
        if (jv1) atomicMin(&S.colmin[j0 + tj_n], __float_as_uint(fminf(acc[1], iv1 ? acc[3] : acc[1])));
      }
      __syncthreads();
    }
    // fold this set-row block: H_v part = max over its rows of the column minima
    if (warp == 0) {
      float cm = lane < rowsv ? __uint_as_float(S.colmin[lane]) : 0.0f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
      S.colmin[lane] = 0x7f800000u;
      if (lane == 0) S.hv = fmaxf(S.hv, cm);
    }
    if (nw_ != w) {  // candidate done: H^2 = max(max_q min_v D^2, max_v min_q D^2) (or MeanMin / Min)
      __syncthreads();
      float hq = 0.0f, sq = 0.0f, mn = __int_as_float(0x7f800000);
      for (int i = tid; i < mq; i += blockDim.x) {
        const float r = __uint_as_float(S.rowmin[i]);
        hq = fmaxf(hq, r);
        sq += sqrtf(r);
        mn = fminf(mn, r);
        S.rowmin[i] = 0x7f800000u;
      }
      float val;
      if (metric == 1) val = block_sum_f(sq, bred) / static_cast<float>(mq);  // MeanMin (a distance)
      else if (metric == 2) val = -block_max_f(-mn, bred);                     // Min (squared)
      else val = fmaxf(block_max_f(hq, bred), S.hv);                          // Hausdorff (squared)
      if (tid == 0) {
        ex[w] = val;
        S.hv = 0.0f;
      }
    }
    __syncthreads();  // (the next iteration's prefetch overwrites this buffer)
    w = nw_;
    vb = nvb;
    buf ^= 1;
  }
  }  // (CTA path)
  }  // (!SMALL)
  __syncthreads();
  if (prof) pt3 = clock64();
  // ---- 3. the k smallest by (exact H^2, id)
  if (nw <= kTxCache) {  // one pass: every window entry's rank among the (distance, id) keys (unique ids)
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(S.jv0);  // row ranges are done with
    for (int x = tid; x < nw; x += blockDim.x)
      keys[x] = (static_cast<unsigned long long>(__float_as_uint(ex[x])) << 32) | static_cast<uint32_t>(cq[win[x]]);
    __syncthreads();
    int64_t* oi = out_ids + static_cast<int64_t>(q) * k;
    float* od = out_dist + static_cast<int64_t>(q) * k;
    for (int x = tid; x < nw; x += blockDim.x) {
      const unsigned long long kx = keys[x];
      int rank = 0;
      for (int y = 0; y < nw; ++y) rank += keys[y] < kx ? 1 : 0;
      if (rank < k) {
        const float e = __uint_as_float(static_cast<uint32_t>(kx >> 32));
        oi[rank] = static_cast<int64_t>(static_cast<uint32_t>(kx & 0xffffffffull));
        od[rank] = metric == 1 ? e : sqrtf(e);
      }
    }
    for (int r = nw + tid; r < k; r += blockDim.x) {
      oi[r] = -1;
      od[r] = __int_as_float(0x7f800000);
    }
    if (prof && tid == 0) {
      const long long pt4 = clock64();
      atomicAdd(&g_k6prof[0], static_cast<unsigned long long>(pt1 - pt0));
      atomicAdd(&g_k6prof[1], static_cast<unsigned long long>(pt2 - pt1));
      atomicAdd(&g_k6prof[2], static_cast<unsigned long long>(pt3 - pt2));
      atomicAdd(&g_k6prof[3], static_cast<unsigned long long>(pt4 - pt3));
      atomicAdd(&g_k6prof[4], 1ull);
      atomicAdd(&g_k6prof[5], static_cast<unsigned long long>(nw));
    }
    return;
  }
  for (int r = 0; r < k; ++r) {
    unsigned long long best = ~0ull;
    for (int x = tid; x < nw; x += blockDim.x) {
      const float e = ex[x];
      if (e < 0.0f) continue;  // taken
      const uint32_t gid = static_cast<uint32_t>(cq[win[x]]);
      const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(e)) << 32) | gid;
      best = key < best ? key : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
      best = t < best ? t : best;
    }
    if (tid == 0) S.best = ~0ull;
    __syncthreads();
    if (lane == 0) atomicMin(&S.best, best);
    __syncthreads();
    const unsigned long long b = S.best;
    if (tid == 0) {
      int64_t* oi = out_ids + static_cast<int64_t>(q) * k;
      float* od = out_dist + static_cast<int64_t>(q) * k;
      if (b == ~0ull) {
        oi[r] = -1;
        od[r] = __int_as_float(0x7f800000);
      } else {
        oi[r] = static_cast<int64_t>(static_cast<uint32_t>(b & 0xffffffffull));
        const float e = __uint_as_float(static_cast<uint32_t>(b >> 32));
        od[r] = metric == 1 ? e : sqrtf(e);
      }
    }
    if (b != ~0ull) {  // mark the winner as taken
      const uint32_t gid = static_cast<uint32_t>(b & 0xffffffffull);
      for (int x = tid; x < nw; x += blockDim.x)
        if (static_cast<uint32_t>(cq[win[x]]) == gid) ex[x] = -1.0f;
    }
    __syncthreads();
  }
}

size_t topk_smem_bytes(int T) { return static_cast<size_t>(T) * 12; }

// shared memory of topk_exact_kernel: RB query rows, two buffers of RBV set rows, the partial sums
static size_t tx_smem(int stride4, int RB, int RBV) {
  return (static_cast<size_t>(RB + 2 * RBV) * stride4 + kTxThreads) * 16;
}

int launch_topk_fixup(const float* approx, const int32_t* cand, const int32_t* count, int T, int k, const float* V,
                      const int64_t* off, int64_t id_base, int d, const float* Qv, const int64_t* qoff,
                      const float* qnorm, float vmax2, float c1, float c2, int exact_all, int64_t* out_ids,
                      float* out_dist, int nq, int64_t* fixup_counter, void* scratch /*[nq][T] x 8 B*/, int metric,
                      const float* approx_err, int max_rows, int max_mq, cudaStream_t st) {
  if (nq <= 0) return BVSS_OK;
  if (k > T) BVSS_FAIL(BVSS_EINVAL, "k > T");
  const int d4 = (d + 3) / 4;
  const int stride4 = (d4 & 1) ? d4 + 2 : d4 + 1;  // odd stride in float4: conflict-free row-parallel reads
  // SMALL: the transposed query tile (32 rows), the two groups' two-slot rings of 64 rows x 9 float4, row starts, minima, row map
  const size_t smem_small = static_cast<size_t>(nch_pad(d4)) * 32 * 16 + 2 * 2 * 64 * 9 * 16 + (kTxCache + 1) * 4 +
                            (kSmRm + kSmRows) * 4 + kSmRows;
  static const bool no_small = getenv("BVSS_K6_NOSMALL") != nullptr;  // developer switch: the CTA path only
  if (!no_small && scratch && (d & 3) == 0 && max_rows <= 32 && max_mq <= 32 && smem_small <= 110 * 1024) {
    int32_t* win = static_cast<int32_t*>(scratch);
    float* ex = reinterpret_cast<float*>(win + static_cast<int64_t>(nq) * T);
    auto kfn = topk_exact_kernel<true>;
    BVSS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_small)));
    static const bool kprof = getenv("BVSS_K6_PROF") != nullptr;
    if (kprof) {
      const int one = 1;
      unsigned long long z[8] = {};
      BVSS_CUDA(cudaMemcpyToSymbolAsync(g_k6prof_on, &one, sizeof(int), 0, cudaMemcpyHostToDevice, st));
      BVSS_CUDA(cudaMemcpyToSymbolAsync(g_k6prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, st));
    }
    kfn<<<nq, kTxThreads, smem_small, st>>>(approx, cand, count, T, k, V, off, id_base, d, d4, stride4, 32, 0, Qv, qoff,
                                            qnorm, vmax2, c1, c2, exact_all, win, ex, out_ids, out_dist, fixup_counter,
                                            metric, approx_err);
    if (kprof) {
      unsigned long long h[8];
      BVSS_CUDA(cudaMemcpyFromSymbolAsync(h, g_k6prof, sizeof(h), 0, cudaMemcpyDeviceToHost, st));
      BVSS_CUDA(cudaStreamSynchronize(st));
      const double c = h[4] ? static_cast<double>(h[4]) : 1.0;
      fprintf(stderr, "[k6prof] ctas=%llu nw/q=%.2f cycles/cta: window %.0f setup %.0f jobs %.0f final %.0f; "
              "warp-job cycles/cta %.0f (of 8 x jobs phase)\n", h[4], h[5] / c, h[0] / c, h[1] / c, h[2] / c,
              h[3] / c, h[6] / c);
    }
    return post_launch("topk_exact_kernel", st);
  }
  int RB = 32, RBV = 16;  // query rows per block; set rows per (double-buffered) block
  while (RB > 4 && tx_smem(stride4, RB, RBV) > 110 * 1024) {  // two CTAs per SM
    if (RBV > 4) RBV >>= 1;
    else RB >>= 1;
  }
  if (scratch && tx_smem(stride4, RB, RBV) <= 110 * 1024) {
    const size_t smem = tx_smem(stride4, RB, RBV);
    int32_t* win = static_cast<int32_t*>(scratch);
    float* ex = reinterpret_cast<float*>(win + static_cast<int64_t>(nq) * T);
    auto kfn = topk_exact_kernel<false>;
    BVSS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kfn<<<nq, kTxThreads, smem, st>>>(approx, cand, count, T, k, V, off, id_base, d, d4, stride4, RB, RBV, Qv,
                                                    qoff, qnorm, vmax2, c1, c2, exact_all, win, ex, out_ids, out_dist,
                                                    fixup_counter, metric, approx_err);
    BVSS_TRY(post_launch("topk_exact_kernel", st));
    return BVSS_OK;
  }
  // very wide vectors: the warp-per-candidate kernel (global-memory operands; Hausdorff only)
  if (metric != 0) BVSS_FAIL(BVSS_EUNSUPPORTED, "MeanMin / Min rerank needs d <= ~3500 (CTA fix-up kernel)");
  const size_t smem = topk_smem_bytes(T);
  if (smem > 190 * 1024) BVSS_FAIL(BVSS_EUNSUPPORTED, "T=%d exceeds the top-k kernel limit (16384)", T);
  if (d % 4 == 0) {
    auto kfn = topk_fixup_kernel<true>;
    BVSS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kfn<<<nq, kTopkThreads, smem, st>>>(approx, cand, count, T, k, V, off, id_base, d, Qv, qoff, qnorm, vmax2, c1, c2,
                                        exact_all, out_ids, out_dist, fixup_counter);
  } else {
    auto kfn = topk_fixup_kernel<false>;
    BVSS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kfn<<<nq, kTopkThreads, smem, st>>>(approx, cand, count, T, k, V, off, id_base, d, Qv, qoff, qnorm, vmax2, c1, c2,
                                        exact_all, out_ids, out_dist, fixup_counter);
  }
  BVSS_TRY(post_launch(__func__, st));
  return BVSS_OK;
}

// ------------------------------------------------------------------- K7 --
__global__ void merge_topk_kernel(const int64_t* __restrict__ ids, const float* __restrict__ dist, int P, int64_t nq,
                                  int k, int64_t* __restrict__ out_ids, float* __restrict__ out_dist) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= nq) return;
  int pos[16];
  for (int p = 0; p < P; ++p) pos[p] = 0;
  for (int r = 0; r < k; ++r) {
    int bp = -1;
    float bd = 0.0f;
    int64_t bi = 0;
    for (int p = 0; p < P; ++p) {
      if (pos[p] >= k) continue;
      const int64_t o = (static_cast<int64_t>(p) * nq + q) * k + pos[p];
      const int64_t id = ids[o];
      if (id < 0) continue;
      const float dd = dist[o];
      if (bp < 0 || dd < bd || (dd == bd && id < bi)) {
        bp = p;
        bd = dd;
        bi = id;
      }
    }
    if (bp < 0) {
      out_ids[q * k + r] = -1;
      out_dist[q * k + r] = __int_as_float(0x7f800000);
    } else {
      out_ids[q * k + r] = bi;
      out_dist[q * k + r] = bd;
      ++pos[bp];
    }
  }
}

int launch_merge_topk(const int64_t* ids, const float* dist, int P, int64_t nq, int k, int64_t* out_ids,
                      float* out_dist, cudaStream_t st) {
  if (P > 16) BVSS_FAIL(BVSS_EUNSUPPORTED, "merge of more than 16 shards");
  if (nq <= 0) return BVSS_OK;
  merge_topk_kernel<<<static_cast<int>(ceil_div<int64_t>(nq, 128)), 128, 0, st>>>(ids, dist, P, nq, k, out_ids, out_dist);
  BVSS_TRY(post_launch(__func__, st));
  return BVSS_OK;
}

}  // namespace bvss
