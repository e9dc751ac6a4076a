// scan.cu — K3: the candidate filter scan (Alg 6 lines 10-13) over
// ALL n database sketches (stage 1 open, reading R6), for a tile of QT query
// sketches held in shared memory.
//   binary: a = popc(S_Q AND S_i);  Hamming = p_Q + p_i - 2a       (reading R1)
//   count : dot = <C_Q, C_i> (dp4a);  L2^2 = |C_Q|^2 + |C_i|^2 - 2dot (reading R2)
// One thread per database set; the DB sketches are streamed chunk-major with
// fully coalesced 16-byte non-allocating loads (every chunk of a set is read
// once per query tile); the query tile is a shared-memory broadcast.  Scores are
// written as keys[q][i] (uint16 for binary, uint32 for count) for K4.
#include "common.cuh"

namespace bvss {

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int QT, int CM>  // CM: 16-byte chunks per sketch (compile-time, = R4/4)
__global__ void __launch_bounds__(256) scan_binary_kernel(const uint4* __restrict__ S, const int32_t* __restrict__ pS,
                                                          int64_t n, int64_t n_stride,
                                                          const uint4* __restrict__ SQ /*[nq][CM] chunks*/,
                                                          const int32_t* __restrict__ pQ, int nq,
                                                          uint16_t* __restrict__ keys, int64_t key_stride) {
  __shared__ uint4 sq[QT][CM];
  __shared__ int spq[QT];
  const int qg = blockIdx.y * QT;
  for (int t = threadIdx.x; t < QT * CM; t += blockDim.x) {
    const int q = t / CM, c = t % CM;
    sq[q][c] = (qg + q < nq) ? SQ[static_cast<int64_t>(qg + q) * CM + c] : make_uint4(0, 0, 0, 0);
  }
  if (threadIdx.x < QT) spq[threadIdx.x] = (qg + threadIdx.x < nq) ? pQ[qg + threadIdx.x] : 0;
  __syncthreads();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint4 a[CM];
#pragma unroll
    for (int c = 0; c < CM; ++c) a[c] = ldg_stream(S + c * n_stride + i);
    const int pi = pS[i];
#pragma unroll
    for (int q = 0; q < QT; ++q) {
      int acc = 0;
#pragma unroll
      for (int c = 0; c < CM; ++c) {
        const uint4 b = sq[q][c];
        acc += __popc(a[c].x & b.x) + __popc(a[c].y & b.y) + __popc(a[c].z & b.z) + __popc(a[c].w & b.w);
      }
      if (qg + q < nq) keys[static_cast<int64_t>(qg + q) * key_stride + i] = static_cast<uint16_t>(spq[q] + pi - 2 * acc);
    }
  }
}

// L1 = false: squared L2 |C_Q|^2 + |C_i|^2 - 2 <C_Q, C_i> (R2); L1 = true: sum_j |C_Q[j] - C_i[j]| (R26),
// per byte |a - b| by vabsdiffu4 and the byte sum by dp4a with ones
template <int QT, bool L1>
__global__ void __launch_bounds__(256) scan_count_kernel(const uint4* __restrict__ C, const int32_t* __restrict__ nC,
                                                         int64_t n, int64_t n_stride, int chunks,
                                                         const uint4* __restrict__ CQ /*[nq][chunks]*/,
                                                         const int32_t* __restrict__ nQ, int nq,
                                                         uint32_t* __restrict__ keys, int64_t key_stride) {
  extern __shared__ uint4 sqc[];  // [QT][chunks]
  __shared__ uint32_t snq[QT];
  const int qg = blockIdx.y * QT;
  for (int t = threadIdx.x; t < QT * chunks; t += blockDim.x) {
    const int q = t / chunks, c = t % chunks;
    sqc[t] = (qg + q < nq) ? CQ[static_cast<int64_t>(qg + q) * chunks + c] : make_uint4(0, 0, 0, 0);
  }
  if (threadIdx.x < QT) snq[threadIdx.x] = (qg + threadIdx.x < nq) ? static_cast<uint32_t>(nQ[qg + threadIdx.x]) : 0u;
  __syncthreads();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t acc[QT];
#pragma unroll
    for (int q = 0; q < QT; ++q) acc[q] = 0u;
#pragma unroll 4
    for (int c = 0; c < chunks; ++c) {
      const uint4 a = ldg_stream(C + c * n_stride + i);
#pragma unroll
      for (int q = 0; q < QT; ++q) {
        const uint4 b = sqc[q * chunks + c];
        if (L1) {
          acc[q] = __dp4a(__vabsdiffu4(a.x, b.x), 0x01010101u, acc[q]);
          acc[q] = __dp4a(__vabsdiffu4(a.y, b.y), 0x01010101u, acc[q]);
          acc[q] = __dp4a(__vabsdiffu4(a.z, b.z), 0x01010101u, acc[q]);
          acc[q] = __dp4a(__vabsdiffu4(a.w, b.w), 0x01010101u, acc[q]);
        } else {
          acc[q] = __dp4a(a.x, b.x, acc[q]);
          acc[q] = __dp4a(a.y, b.y, acc[q]);
          acc[q] = __dp4a(a.z, b.z, acc[q]);
          acc[q] = __dp4a(a.w, b.w, acc[q]);
        }
      }
    }
    const uint32_t ni = static_cast<uint32_t>(nC[i]);
#pragma unroll
    for (int q = 0; q < QT; ++q)
      if (qg + q < nq) keys[static_cast<int64_t>(qg + q) * key_stride + i] = L1 ? acc[q] : snq[q] + ni - 2u * acc[q];
  }
}

int launch_scan(int kind, const void* S, const int32_t* mass, int64_t n, int64_t n_stride, int m, const void* SQ,
                const int32_t* massQ, int nq, void* keys, int64_t key_stride, int num_sms, cudaStream_t st) {
  if (nq <= 0 || n <= 0) return BVSS_OK;
  const int blocks_x_full = static_cast<int>(ceil_div<int64_t>(n, 256));
  if (kind == BVSS_SKETCH_BINARY) {
    constexpr int QT = 8;
    const int R4 = ((m / 32) + 3) & ~3;
    const int CM = R4 / 4;
    const int gy = ceil_div(nq, QT);
    // enough CTAs for ~4 waves of 148 SMs x 8 resident CTAs, each thread looping over sets
    int gx = blocks_x_full;
    const int cap = ceil_div(num_sms * 8 * 4, gy);
    if (gx > cap) gx = cap < 1 ? 1 : cap;
    dim3 grid(gx, gy);
    const uint4* Sv = static_cast<const uint4*>(S);
    const uint4* Qv = static_cast<const uint4*>(SQ);
    uint16_t* K = static_cast<uint16_t*>(keys);
    switch (CM) {
#define BVSS_SCAN_CASE(c) \
  case c: scan_binary_kernel<QT, c><<<grid, 256, 0, st>>>(Sv, mass, n, n_stride, Qv, massQ, nq, K, key_stride); break;
      BVSS_SCAN_CASE(1) BVSS_SCAN_CASE(2) BVSS_SCAN_CASE(3) BVSS_SCAN_CASE(4) BVSS_SCAN_CASE(5) BVSS_SCAN_CASE(6)
      BVSS_SCAN_CASE(7) BVSS_SCAN_CASE(8) BVSS_SCAN_CASE(9) BVSS_SCAN_CASE(10) BVSS_SCAN_CASE(11) BVSS_SCAN_CASE(12)
      BVSS_SCAN_CASE(13) BVSS_SCAN_CASE(14) BVSS_SCAN_CASE(15) BVSS_SCAN_CASE(16)
#undef BVSS_SCAN_CASE
      default: BVSS_FAIL(BVSS_EUNSUPPORTED, "binary scan: m=%d too large", m);
    }
  } else {
    constexpr int QT = 8;
    const int chunks = m / 16;
    const int gy = ceil_div(nq, QT);
    int gx = blocks_x_full;
    const int cap = ceil_div(num_sms * 8 * 4, gy);
    if (gx > cap) gx = cap < 1 ? 1 : cap;
    const size_t smem = static_cast<size_t>(QT) * chunks * 16;
    auto kfn = kind == 2 ? scan_count_kernel<QT, true> : scan_count_kernel<QT, false>;  // kind 2: count, L1
    BVSS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kfn<<<dim3(gx, gy), 256, smem, st>>>(static_cast<const uint4*>(S), mass, n, n_stride, chunks,
                                         static_cast<const uint4*>(SQ), massQ, nq, static_cast<uint32_t*>(keys),
                                         key_stride);
  }
  BVSS_TRY(post_launch(__func__, st));
  return BVSS_OK;
}

}  // namespace bvss
