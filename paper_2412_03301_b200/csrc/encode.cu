// encode.cu — K1: FlyHash projection + winner-take-all (Def 7, PAPER.md P:317-320;
// Alg 1 lines 4-7), fused with the refine-operand preparation (K9:
// fp32 squared norm and the scaled fp16 hi/lo split of every vector).
//
// One warp per vector.  The vector is staged in shared memory; lane l computes
// the activations of rows j = l + 32 t (t < m/32) as a left-to-right fp32 sum
// over W's sorted index list starting from +0.0f (reading R8), so codes are
// bit-identical to the oracle.  The L-th largest activation is found by a
// 32-step bisection on order-preserving uint32 keys (warp redux counts), ties
// at the threshold go to the lowest row index (reading R4), and code word t is
// a warp ballot, so the code is written without any shared-memory scatter.
#include "common.cuh"

namespace bvss {

template <int RM, int SS>  // RM = capacity in 32-row groups (m/32 <= RM); SS = s when fixed at compile time, else 0
__global__ void __launch_bounds__(256) flyhash_wta_kernel(
    const float* __restrict__ V, int64_t nvec, int d, const uint16_t* __restrict__ Wt /*[s][m]*/, int m,
    int s, int L, uint32_t* __restrict__ codes /*[nvec][m/32] or null*/, float* __restrict__ norms /*[nvec] or null*/,
    __half* __restrict__ hs, __half* __restrict__ ls /*[KS][rows/8][KCS][8][64] or null*/, float* __restrict__ scale,
    int dpad, int64_t rows, const int64_t* __restrict__ dst_row, int kcs) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint16_t* sW = reinterpret_cast<uint16_t*>(smem);
  float* sV = reinterpret_cast<float*>(smem + ((static_cast<size_t>(s) * m * 2 + 15) & ~size_t(15)));
  for (int i = threadIdx.x; i < s * m; i += blockDim.x) sW[i] = Wt[i];
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  float* myv = sV + static_cast<size_t>(warp) * d;
  const int R = m >> 5;
  constexpr int MW = (RM + 31) / 32;

  for (int64_t vi = static_cast<int64_t>(blockIdx.x) * nwarps + warp; vi < nvec;
       vi += static_cast<int64_t>(gridDim.x) * nwarps) {
    const float* src = V + vi * d;
    float nrm = 0.0f;
    for (int i = lane; i < d; i += 32) {
      float x = src[i];
      myv[i] = x;
      nrm = __fmaf_rn(x, x, nrm);
    }
    if (hs != nullptr) {
      // scale: s = 2^e with max|x| <= s (exact power-of-two scaling), y = x / s in [-1, 1]
      float mx = 0.0f;
      for (int i = lane; i < d; i += 32) mx = fmaxf(mx, fabsf(myv[i]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      int ex = 0;
      if (mx > 0.0f) frexpf(mx, &ex);  // mx = f 2^ex, f in [0.5, 1)
      const float inv = ldexpf(1.0f, -ex);
      // super-chunk-major, pre-swizzled (refine.cu): element i of row `row` goes to 128-byte K-chunk
      // kc = i/64 (super kc/KCS, slot kc%KCS) of its 8-row group, 16-byte unit ((i%64)/8) ^ (row%8)
      const int64_t row = dst_row ? dst_row[vi] : vi;
      const int64_t groups = rows >> 3;
      if (lane == 0) scale[row] = ldexpf(1.0f, ex);
      for (int i = lane; i < dpad; i += 32) {
        const float y = i < d ? myv[i] * inv : 0.0f;
        const __half h = __float2half_rn(y);
        const __half l = __float2half_rn(y - __half2float(h));
        const int kc = i >> 6, u = (i >> 3) & 7, e = i & 7;
        const int ks = kc / kcs, kq = kc % kcs;
        const int64_t o = ((((static_cast<int64_t>(ks) * groups + (row >> 3)) * kcs + kq) * 8 + (row & 7)) << 6) +
                          ((u ^ static_cast<int>(row & 7)) << 3) + e;
        hs[o] = h;
        if (ls != nullptr) ls[o] = l;  // the lo piece only for the 3-term Gram (refine_terms = 3)
      }
    }
    if (norms != nullptr) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
      if (lane == 0) norms[vi] = nrm;
    }
    __syncwarp();
    if (codes != nullptr) {
      uint32_t key[RM];
#pragma unroll
      for (int t = 0; t < RM; ++t) {
        key[t] = 0u;  // rows >= m never win: every real key is > 0
        if (t < R) {
          const int j = t * 32 + lane;
          float acc = 0.0f;
          if (SS > 0) {  // all s index loads and gathers issue together; only the adds are chained
            float g[SS > 0 ? SS : 1];
#pragma unroll
            for (int u = 0; u < SS; ++u) g[u] = myv[sW[u * m + j]];
#pragma unroll
            for (int u = 0; u < SS; ++u) acc = __fadd_rn(acc, g[u]);
          } else {
            for (int u = 0; u < s; ++u) acc = __fadd_rn(acc, myv[sW[u * m + j]]);
          }
          key[t] = float_order_key(acc);
        }
      }
      // largest K with |{j : key_j >= K}| >= L  (the L-th largest key)
      uint32_t prefix = 0u;
#pragma unroll 1
      for (int b = 31; b >= 0; --b) {
        const uint32_t cand = prefix | (1u << b);
        int cnt = 0;
#pragma unroll
        for (int t = 0; t < RM; ++t) cnt += key[t] >= cand ? 1 : 0;
        if (warp_sum(cnt) >= L) prefix = cand;
      }
      int gt = 0;
#pragma unroll
      for (int t = 0; t < RM; ++t) gt += key[t] > prefix ? 1 : 0;
      int need = L - warp_sum(gt);
      uint32_t mw[MW];
#pragma unroll
      for (int i = 0; i < MW; ++i) mw[i] = 0u;
#pragma unroll
      for (int t = 0; t < RM; ++t) {
        if (t < R) {
          uint32_t w = __ballot_sync(0xffffffffu, key[t] > prefix);
          uint32_t eq = __ballot_sync(0xffffffffu, key[t] == prefix);
          if (need > 0 && eq != 0u) {
            const int c = __popc(eq);
            if (c <= need) {
              w |= eq;
              need -= c;
            } else {  // the `need` lowest rows among the ties
              uint32_t e = eq;
              for (int i = 0; i < need; ++i) e &= e - 1u;  // drop the lowest `need` bits
              w |= eq & ~e;
              need = 0;
            }
          }
          if ((t & 31) == lane) mw[t >> 5] = w;
        }
      }
#pragma unroll
      for (int i = 0; i < MW; ++i) {
        const int wd = lane + 32 * i;
        if (wd < R) codes[vi * R + wd] = mw[i];
      }
    }
    __syncwarp();
  }
}

size_t encode_smem_bytes(int m, int s, int d) {
  return ((static_cast<size_t>(s) * m * 2 + 15) & ~size_t(15)) + static_cast<size_t>(8) * d * 4;
}

int launch_encode(const float* V, int64_t nvec, int d, const uint16_t* Wt, int m, int s, int L, uint32_t* codes,
                  float* norms, __half* hs, __half* ls, float* scale, int dpad, int64_t rows, const int64_t* dst_row,
                  int kcs, int num_sms, cudaStream_t st) {
  if (nvec <= 0) return BVSS_OK;
  const size_t smem = encode_smem_bytes(m, s, d);
  const int R = m / 32;
  const int64_t want = ceil_div<int64_t>(nvec, 8);
  const int grid = static_cast<int>(want < int64_t(num_sms) * 8 ? want : int64_t(num_sms) * 8);
#define BVSS_ENC(RMv)                                                                                     \
  do {                                                                                                    \
    auto kfn = s == 8 ? flyhash_wta_kernel<RMv, 8> : s == 6 ? flyhash_wta_kernel<RMv, 6>                  \
             : s == 12 ? flyhash_wta_kernel<RMv, 12> : flyhash_wta_kernel<RMv, 0>;                        \
    BVSS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem))); \
    kfn<<<grid, 256, smem, st>>>(V, nvec, d, Wt, m, s, L, codes, norms, hs, ls, scale, dpad, rows, dst_row, kcs); \
  } while (0)
  if (R <= 16) BVSS_ENC(16);
  else if (R <= 32) BVSS_ENC(32);
  else if (R <= 64) BVSS_ENC(64);
  else BVSS_FAIL(BVSS_EUNSUPPORTED, "m=%d exceeds the 2048-row encoder limit", m);
#undef BVSS_ENC
  BVSS_TRY(post_launch(__func__, st));
  return BVSS_OK;
}

// ------------------------------------------------------------- validation --
__global__ void finite_check_kernel(const float* __restrict__ x, int64_t count, int* __restrict__ bad) {
  int any = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    any |= !isfinite(x[i]);
  if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(bad, 1);
}

int launch_finite_check(const float* x, int64_t count, int* bad_dev, int num_sms, cudaStream_t st) {
  if (count <= 0) return BVSS_OK;
  finite_check_kernel<<<num_sms * 4, 256, 0, st>>>(x, count, bad_dev);
  BVSS_TRY(post_launch(__func__, st));
  return BVSS_OK;
}

}  // namespace bvss
