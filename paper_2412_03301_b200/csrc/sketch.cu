// sketch.cu — K2: per-set sketches over the segmented (set_offsets) layout, one
// warp per set.
//   binary  : S = OR of the set's codes   (Def 10, Alg 5 lines 3-5)
//   count   : C = sum of the set's codes  (Def 8, Alg 3 line 4), uint8
//             saturating at 255 (reading R14)
// plus the per-set mass used by the scan: popc(S) (binary) or ||C||^2 (count).
//
// Scan layout: sketches are stored chunk-major so that a
// thread-per-set scan issues fully coalesced 16-byte loads:
//   binary: uint4  [R4/4][n]  (R4 = m/32 rounded up to 4 words; zero padded)
//   count : uint4  [m/16][n]  (16 counters per chunk)
#include "common.cuh"

namespace bvss {

template <int WM>  // words per lane capacity: m/32 <= 32*WM
__global__ void __launch_bounds__(256) sketch_binary_kernel(const uint32_t* __restrict__ codes, int R,
                                                            const int64_t* __restrict__ off, int64_t n,
                                                            uint32_t* __restrict__ S,
                                                            int32_t* __restrict__ mass, int64_t cstride,
                                                            int64_t sstride) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int R4 = (R + 3) & ~3;
  for (int64_t set = w0; set < n; set += nw) {
    uint32_t acc[WM];
#pragma unroll
    for (int i = 0; i < WM; ++i) acc[i] = 0u;
    const int64_t b = off[set], e = off[set + 1];
    for (int64_t v = b; v < e; ++v) {
#pragma unroll
      for (int i = 0; i < WM; ++i) {
        const int wd = lane + 32 * i;
        if (wd < R) acc[i] |= codes[v * R + wd];
      }
    }
    int p = 0;
#pragma unroll
    for (int i = 0; i < WM; ++i) {
      const int wd = lane + 32 * i;
      if (wd < R4) {
        p += __popc(acc[i]);
        S[((static_cast<int64_t>(wd >> 2) * cstride + set * sstride) << 2) + (wd & 3)] = wd < R ? acc[i] : 0u;
      }
    }
    p = warp_sum(p);
    if (lane == 0) mass[set] = p;
  }
}

template <int WM>
__global__ void __launch_bounds__(256) sketch_count_kernel(const uint32_t* __restrict__ codes, int R,
                                                           const int64_t* __restrict__ off, int64_t n,
                                                           uint4* __restrict__ C,
                                                           int32_t* __restrict__ mass, int64_t cstride,
                                                           int64_t sstride) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t set = w0; set < n; set += nw) {
    // lane owns words lane + 32 i; 8 packed uint8x4 counters per word (saturating adds)
    uint32_t cnt[WM][8];
#pragma unroll
    for (int i = 0; i < WM; ++i)
#pragma unroll
      for (int g = 0; g < 8; ++g) cnt[i][g] = 0u;
    const int64_t b = off[set], e = off[set + 1];
    for (int64_t v = b; v < e; ++v) {
#pragma unroll
      for (int i = 0; i < WM; ++i) {
        const int wd = lane + 32 * i;
        if (wd < R) {
          const uint32_t x = codes[v * R + wd];
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            const uint32_t nib = (x >> (4 * g)) & 0xFu;
            cnt[i][g] = __vaddus4(cnt[i][g], (nib * 0x00204081u) & 0x01010101u);
          }
        }
      }
    }
    uint32_t sq = 0u;
#pragma unroll
    for (int i = 0; i < WM; ++i) {
      const int wd = lane + 32 * i;
      if (wd < R) {
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const uint32_t c = cnt[i][g];
          sq += __dp4a(c, c, 0u);
        }
        // word wd = counters 32wd .. 32wd+31 = 16-byte chunks 2wd and 2wd+1
        C[static_cast<int64_t>(2 * wd) * cstride + set * sstride] = make_uint4(cnt[i][0], cnt[i][1], cnt[i][2], cnt[i][3]);
        C[static_cast<int64_t>(2 * wd + 1) * cstride + set * sstride] =
            make_uint4(cnt[i][4], cnt[i][5], cnt[i][6], cnt[i][7]);
      }
    }
    sq = static_cast<uint32_t>(warp_sum(static_cast<int>(sq)));
    if (lane == 0) mass[set] = static_cast<int32_t>(sq);
  }
}

// Layout of S in 16-byte chunks: chunk c of set i at c * cstride + i * sstride.
//   scan (chunk-major): cstride = n, sstride = 1;  row-major: cstride = 1, sstride = chunks per set.
int launch_sketch(const uint32_t* codes, int m, const int64_t* off, int64_t n, int kind, void* S, int32_t* mass,
                  int64_t cstride, int64_t sstride, int num_sms, cudaStream_t st) {
  if (n <= 0) return BVSS_OK;
  const int R = m / 32;
  const int64_t want = ceil_div<int64_t>(n, 8);
  const int grid = static_cast<int>(want < int64_t(num_sms) * 16 ? want : int64_t(num_sms) * 16);
  if (kind == BVSS_SKETCH_BINARY) {
    if (R <= 32)
      sketch_binary_kernel<1><<<grid, 256, 0, st>>>(codes, R, off, n, static_cast<uint32_t*>(S), mass, cstride, sstride);
    else if (R <= 64)
      sketch_binary_kernel<2><<<grid, 256, 0, st>>>(codes, R, off, n, static_cast<uint32_t*>(S), mass, cstride, sstride);
    else
      BVSS_FAIL(BVSS_EUNSUPPORTED, "m=%d too large", m);
  } else {
    if (R <= 32)
      sketch_count_kernel<1><<<grid, 256, 0, st>>>(codes, R, off, n, static_cast<uint4*>(S), mass, cstride, sstride);
    else if (R <= 64)
      sketch_count_kernel<2><<<grid, 256, 0, st>>>(codes, R, off, n, static_cast<uint4*>(S), mass, cstride, sstride);
    else
      BVSS_FAIL(BVSS_EUNSUPPORTED, "m=%d too large", m);
  }
  BVSS_TRY(post_launch(__func__, st));
  return BVSS_OK;
}

// chunked -> row-major (exports and query sketches)
__global__ void unchunk_kernel(const uint32_t* __restrict__ S, int64_t n_stride, int64_t first, int64_t count,
                               int words /*row-major words per set*/, int chunk_words /*4*/, uint32_t* __restrict__ out) {
  const int64_t total = count * words;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / words;
    const int w = static_cast<int>(t % words);
    out[t] = S[((w / chunk_words) * n_stride + first + r) * chunk_words + (w % chunk_words)];
  }
}

int launch_unchunk(const void* S, int64_t n_stride, int64_t first, int64_t count, int words, uint32_t* out,
                   cudaStream_t st) {
  if (count <= 0) return BVSS_OK;
  unchunk_kernel<<<256, 256, 0, st>>>(static_cast<const uint32_t*>(S), n_stride, first, count, words, 4, out);
  BVSS_TRY(post_launch(__func__, st));
  return BVSS_OK;
}

}  // namespace bvss
