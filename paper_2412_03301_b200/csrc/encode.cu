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
#include <cstdlib>

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
      // largest K with |{j : key_j >= K}| >= L  (the L-th largest key).  The bisection stops as soon as exactly
      // L keys are >= the candidate: the winners are then exactly those keys (every other key is below it), so
      // the lower bits of K do not matter -- for continuous activations the L-th and (L+1)-th keys part after
      // the sign, the exponent and a few mantissa bits (~16 steps instead of 32).  Identical codes; cfg3 build
      // 72-111 -> 63-65 ms for 7.2M vectors (profiles/r02/s3/encoder_builds_ab.log)
      uint32_t prefix = 0u;
#pragma unroll 1
      for (int b = 31; b >= 0; --b) {
        const uint32_t cand = prefix | (1u << b);
        int cnt = 0;
#pragma unroll
        for (int t = 0; t < RM; ++t) cnt += key[t] >= cand ? 1 : 0;
        const int c = warp_sum(cnt);
        if (c >= L) prefix = cand;
        if (c == L) break;
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

// ---------------------------------------------------------------------------------------------------------
// K1, lane-per-vector form (codes only).  A warp encodes 32 vectors at once, lane = vector: the tile is staged
// dim-major in shared memory ([d][32] fp32, column = vector ^ (dim & 31), so both the transposing stores and
// the gathers are conflict-free), W's row j is a warp-uniform list of s indices (a broadcast), and each gather
// serves 32 vectors with one conflict-free wavefront (the warp-per-vector form's gathers at 32 random
// addresses collide ~3.5-way and need a W-index load each).  The additions are the same left-to-right fp32
// sums from +0.0f over the sorted S_j (reading R8), so the activations are bit-identical.
// WTA per lane: rows come in increasing j; a row enters the lane's candidate buffer (shared memory, column =
// lane) when its key beats the lane's threshold theta (strictly: a later row loses every tie, reading R4);
// when a buffer nears its capacity it is compacted to the exact top L by (key desc, j asc) -- the L-th
// largest key K by bisection on the key bits, every key > K and the first (lowest-j) entries equal to K --
// and theta = K.  Dropped rows can never re-enter the top L, so the final compaction is exactly Def 7's WTA.
constexpr int kLanesRB = 8;  // rows per block between buffer checks

__device__ __forceinline__ int lanes_compact(uint32_t* kb, uint16_t* jb, int cnt, int L, int lane, uint32_t* theta) {
  const int cmax = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(cnt));
  uint32_t kmin = 0xffffffffu, kmax = 0u;
  for (int e = 0; e < cmax; ++e)
    if (e < cnt) {
      const uint32_t k = kb[e * 32 + lane];
      kmin = min(kmin, k);
      kmax = max(kmax, k);
    }
  const bool act = cnt > L;
  // bisection below the lane's common high bits of kmin / kmax; the loop bound is the warp's widest span
  const uint32_t diff = act ? (kmin ^ kmax) : 0u;
  const int hb = diff ? 31 - __clz(diff) : -1;
  const int hbw = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(hb + 1))) - 1;
  uint32_t prefix = hb >= 0 ? (kmin & ~((2u << hb) - 1u)) : kmin;  // (hb = 31: the mask is 0)
  if (hb == 31) prefix = 0u;
  for (int b = hbw; b >= 0; --b) {
    const uint32_t cand = prefix | (1u << b);
    int c = 0;
    for (int e = 0; e < cmax; ++e) c += (e < cnt && kb[e * 32 + lane] >= cand) ? 1 : 0;
    if (act && b <= hb && c >= L) prefix = cand;
  }
  if (!act) return cnt;
  int gt = 0;
  for (int e = 0; e < cmax; ++e) gt += (e < cnt && kb[e * 32 + lane] > prefix) ? 1 : 0;
  int need = L - gt, w = 0;
  for (int e = 0; e < cmax; ++e)
    if (e < cnt) {
      const uint32_t k = kb[e * 32 + lane];
      bool keep = k > prefix;
      if (!keep && k == prefix && need > 0) {
        keep = true;
        --need;
      }
      if (keep) {
        const uint16_t j = jb[e * 32 + lane];
        kb[w * 32 + lane] = k;
        jb[w * 32 + lane] = j;
        ++w;
      }
    }
  *theta = prefix;
  return w;
}

template <int SS>
__global__ void __launch_bounds__(128) flyhash_lanes_kernel(const float* __restrict__ V, int64_t nvec, int d,
                                                            const uint16_t* __restrict__ Wt /*[s][m]*/, int m, int L,
                                                            int cap, uint32_t* __restrict__ codes) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int S = SS;
  uint16_t* sW = reinterpret_cast<uint16_t*>(smem);  // [m][S] (row-major: row j's indices are contiguous)
  const size_t wbytes = (static_cast<size_t>(m) * S * 2 + 15) & ~size_t(15);
  const int R = m >> 5;
  const size_t per_warp = static_cast<size_t>(d) * 128 + static_cast<size_t>(cap) * 128 + static_cast<size_t>(cap) * 64 +
                          static_cast<size_t>(R) * 128;
  for (int i = threadIdx.x; i < S * m; i += blockDim.x) {
    const int u = i / m, j = i - u * m;
    sW[j * S + u] = Wt[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  uint8_t* wb = smem + wbytes + per_warp * warp;
  float* sV = reinterpret_cast<float*>(wb);                                         // [d][32]
  uint32_t* kb = reinterpret_cast<uint32_t*>(wb + static_cast<size_t>(d) * 128);     // [cap][32]
  uint16_t* jb = reinterpret_cast<uint16_t*>(wb + static_cast<size_t>(d) * 128 + static_cast<size_t>(cap) * 128);
  uint32_t* cw = reinterpret_cast<uint32_t*>(wb + static_cast<size_t>(d) * 128 + static_cast<size_t>(cap) * 192);  // [R][32]
  const int64_t ntile = (nvec + 31) >> 5;
  for (int64_t tile = static_cast<int64_t>(blockIdx.x) * nwarps + warp; tile < ntile;
       tile += static_cast<int64_t>(gridDim.x) * nwarps) {
    const int64_t v0 = tile << 5;
    const int nv = nvec - v0 < 32 ? static_cast<int>(nvec - v0) : 32;
    __syncwarp();
#pragma unroll 4
    for (int v = 0; v < 32; ++v) {  // dim-major staging (lane = dim within a 32-dim group)
      const float* src = V + (v0 + v) * d;
      for (int c = lane; c < d; c += 32) sV[c * 32 + (v ^ lane)] = v < nv ? src[c] : 0.0f;
    }
    for (int w = 0; w < R; ++w) cw[w * 32 + lane] = 0u;
    __syncwarp();
    uint32_t theta = 0u;  // every real key is > 0
    int cnt = 0;
    for (int j0 = 0; j0 < m; j0 += kLanesRB) {
      uint32_t key[kLanesRB];
#pragma unroll
      for (int i = 0; i < kLanesRB; ++i) {
        // row j's S indices by the widest aligned broadcast loads (S = 8: one 16-byte load)
        uint16_t wr[S];
        if constexpr (S % 8 == 0) {
#pragma unroll
          for (int q = 0; q < S / 8; ++q) *reinterpret_cast<uint4*>(wr + 8 * q) = reinterpret_cast<const uint4*>(sW + (j0 + i) * S)[q];
        } else if constexpr (S % 4 == 0) {
#pragma unroll
          for (int q = 0; q < S / 4; ++q) *reinterpret_cast<uint2*>(wr + 4 * q) = reinterpret_cast<const uint2*>(sW + (j0 + i) * S)[q];
        } else {
#pragma unroll
          for (int q = 0; q < S / 2; ++q) *reinterpret_cast<uint32_t*>(wr + 2 * q) = reinterpret_cast<const uint32_t*>(sW + (j0 + i) * S)[q];
        }
        float g[S];
#pragma unroll
        for (int u = 0; u < S; ++u) {
          const int x = wr[u];
          g[u] = sV[x * 32 + (lane ^ (x & 31))];
        }
        float acc = 0.0f;
#pragma unroll
        for (int u = 0; u < S; ++u) acc = __fadd_rn(acc, g[u]);
        key[i] = float_order_key(acc);
      }
#pragma unroll
      for (int i = 0; i < kLanesRB; ++i)
        if (key[i] > theta) {
          kb[cnt * 32 + lane] = key[i];
          jb[cnt * 32 + lane] = static_cast<uint16_t>(j0 + i);
          ++cnt;
        }
      if (__any_sync(0xffffffffu, cnt > cap - kLanesRB)) cnt = lanes_compact(kb, jb, cnt, L, lane, &theta);
    }
    cnt = lanes_compact(kb, jb, cnt, L, lane, &theta);  // exactly the top L
    for (int e = 0; e < cnt; ++e) {  // (word w of vector `lane` lives at column lane ^ (w & 31))
      const int j = jb[e * 32 + lane], w = j >> 5;
      cw[w * 32 + (lane ^ (w & 31))] |= 1u << (j & 31);
    }
    __syncwarp();
    for (int v = 0; v < nv; ++v)  // code of vector v: word w from lane w (coalesced rows, conflict-free reads)
      for (int w = lane; w < R; w += 32) codes[(v0 + v) * R + w] = cw[w * 32 + (v ^ (w & 31))];
  }
}

// shared memory of the lane-per-vector encoder per warp, and whether it applies (s compiled, cap fits)
static size_t lanes_warp_bytes(int m, int d, int cap) {
  return static_cast<size_t>(d) * 128 + static_cast<size_t>(cap) * 192 + static_cast<size_t>(m / 32) * 128;
}

int launch_encode_lanes(const float* V, int64_t nvec, int d, const uint16_t* Wt, int m, int s, int L,
                        uint32_t* codes, int num_sms, cudaStream_t st, bool* done) {
  *done = false;
  // opt-in (BVSS_ENC_LANES=1): measured slower than the warp-per-vector kernel on B200 (cfg3, 3.6M vectors:
  // build 104 ms vs 37 ms; bit-identical codes): with 64 KB of shared memory per warp only 3 warps fit on an
  // SM and the gather / compaction chains are latency-bound
  const char* env = getenv("BVSS_ENC_LANES");
  if (!env || atoi(env) == 0) return BVSS_OK;
  if (nvec <= 0 || codes == nullptr || m > 65535 || (s != 8 && s != 6 && s != 12)) return BVSS_OK;
  const int cap = ((L + kLanesRB + 24) + 7) & ~7;  // room for 3 blocks of appends past L between compactions
  const size_t wbytes = (static_cast<size_t>(m) * s * 2 + 15) & ~size_t(15);
  const size_t pw = lanes_warp_bytes(m, d, cap);
  int warps = static_cast<int>((227 * 1024 - wbytes) / pw);
  if (warps > 4) warps = 4;
  if (warps < 2) return BVSS_OK;  // (large d / m / L: the warp-per-vector kernel)
  const size_t smem = wbytes + pw * warps;
  const int64_t ntile = (nvec + 31) / 32;
  const int64_t want = ceil_div<int64_t>(ntile, warps);
  const int grid = static_cast<int>(want < num_sms ? want : num_sms);
  auto kfn = s == 8 ? flyhash_lanes_kernel<8> : s == 6 ? flyhash_lanes_kernel<6> : flyhash_lanes_kernel<12>;
  BVSS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kfn<<<grid, 32 * warps, smem, st>>>(V, nvec, d, Wt, m, L, cap, codes);
  BVSS_TRY(post_launch(__func__, st));
  *done = true;
  return BVSS_OK;
}

size_t encode_smem_bytes(int m, int s, int d) {
  return ((static_cast<size_t>(s) * m * 2 + 15) & ~size_t(15)) + static_cast<size_t>(8) * d * 4;
}

int launch_encode(const float* V, int64_t nvec, int d, const uint16_t* Wt, int m, int s, int L, uint32_t* codes,
                  float* norms, __half* hs, __half* ls, float* scale, int dpad, int64_t rows, const int64_t* dst_row,
                  int kcs, int num_sms, cudaStream_t st) {
  if (nvec <= 0) return BVSS_OK;
  bool lanes = false;  // codes by the lane-per-vector kernel; this one then writes only norms and the split
  BVSS_TRY(launch_encode_lanes(V, nvec, d, Wt, m, s, L, codes, num_sms, st, &lanes));
  if (lanes) {
    codes = nullptr;
    if (norms == nullptr && hs == nullptr) return BVSS_OK;
  }
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
