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
#include "common.cuh"

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

size_t topk_smem_bytes(int T) { return static_cast<size_t>(T) * 12; }

int launch_topk_fixup(const float* approx, const int32_t* cand, const int32_t* count, int T, int k, const float* V,
                      const int64_t* off, int64_t id_base, int d, const float* Qv, const int64_t* qoff,
                      const float* qnorm, float vmax2, float c1, float c2, int exact_all, int64_t* out_ids,
                      float* out_dist, int nq, int64_t* fixup_counter, cudaStream_t st) {
  if (nq <= 0) return BVSS_OK;
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
