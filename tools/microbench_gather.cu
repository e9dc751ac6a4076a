// Developer microbenchmark (not part of the library): the refine gather pattern in isolation.
// Persistent CTA per SM; warp 0 issues, per stage, one cp.async.bulk per set (lane-parallel)
// for sets of m in [4, 32] rows drawn at random from a large pool, until the stage holds
// `rows` rows; row bytes R per stage (KCS x 128 B); set slab = pad(m) x R, where pad rounds m
// up to `align` rows; a consumer warp releases the stage when it lands.  Reports useful
// (unpadded) GB/s and copied GB/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_gather microbench_gather.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
               : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) { while (!try_wait(b, ph)) {} }
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void arrive_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(n), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// pool: nsets sets, each occupying a slot of 32 rows x R bytes (so any pad(m) <= 32 fits)
__global__ void gather(const char* pool, size_t nsets, int R, int rows, int align, int S, int iters,
                       unsigned long long* useful, unsigned long long* copied, int* sink) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ uint64_t full[8], empty[8];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t stage_bytes = (uint32_t)rows * R;
  if (threadIdx.x < 32) {
    unsigned long long u = 0, c = 0;
    for (int i = 0; i < iters; ++i) {
      const int s = i % S;
      wait(&empty[s], ((i / S) & 1) ^ 1);
      // lane j draws set j of this stage: m, source; prefix over padded rows decides who fits
      const uint32_t h = hash(blockIdx.x * 7919u + i * 131u + lane);
      const int m = 4 + (int)(h % 29u);
      const int mp = (m + align - 1) / align * align;
      int incl = mp;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const bool fits = incl <= rows;
      const int used = __shfl_sync(0xffffffffu, fits ? incl : 0, 31 - __clz(__ballot_sync(0xffffffffu, fits)));
      const uint32_t tx = (uint32_t)used * R;
      if (lane == 0) arrive_tx(&full[s], tx);
      __syncwarp();
      if (fits) {
        const size_t set = hash(h) % nsets;
        bulk(su32(sm + (size_t)s * stage_bytes + (size_t)(incl - mp) * R), pool + set * 32 * (size_t)R,
             (uint32_t)mp * R, &full[s]);
        u += (unsigned long long)m * R;
        c += (unsigned long long)mp * R;
      }
    }
    for (int o = 16; o; o >>= 1) {
      u += __shfl_xor_sync(0xffffffffu, u, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (lane == 0) { atomicAdd(useful, u); atomicAdd(copied, c); }
  } else if (threadIdx.x == 32) {
    int acc = 0;
    for (int i = 0; i < iters; ++i) {
      const int s = i % S;
      wait(&full[s], (i / S) & 1);
      acc += sm[(size_t)s * stage_bytes];
      arrive(&empty[s]);
    }
    if (acc == 12345) *sink = acc;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)24 << 30;
  char* pool;
  unsigned long long* ctr;
  int* sink;
  cudaMalloc(&pool, total);
  cudaMalloc(&ctr, 16);
  cudaMalloc(&sink, 4);
  cudaMemset(pool, 1, total);
  cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // {R (row bytes per stage), rows per stage, align, stages}
  const int cfgs[][4] = {
      {256, 256, 8, 2}, {256, 256, 1, 2}, {256, 256, 8, 3}, {256, 256, 1, 3},  // KCS = 2
      {128, 256, 8, 4}, {128, 256, 1, 4}, {128, 256, 1, 6},                    // KCS = 1
      {384, 256, 8, 2}, {384, 256, 1, 2},                                      // KCS = 3
      {768, 128, 1, 2}, {768, 96, 1, 3}, {768, 64, 1, 4},                      // whole K (d = 384)
      {512, 128, 1, 3}, {512, 96, 1, 4},
  };
  for (auto& c : cfgs) {
    const int R = c[0], rows = c[1], align = c[2], S = c[3];
    const size_t smem = (size_t)S * rows * R;
    if (smem > 226 * 1024) { printf("skip R=%d rows=%d S=%d\n", R, rows, S); continue; }
    const size_t nsets = total / (32 * (size_t)R);
    const int iters = (int)(((size_t)6 << 30) / sms / ((size_t)rows * R));
    double gu = 0, gc = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(ctr, 0, 16);
      cudaEventRecord(e0);
      gather<<<sms, 64, smem>>>(pool, nsets, R, rows, align, S, iters, ctr, ctr + 1, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long h[2];
      cudaMemcpy(h, ctr, 16, cudaMemcpyDeviceToHost);
      gu = h[0] / ms / 1e6;
      gc = h[1] / ms / 1e6;
    }
    printf("R=%4d rows=%3d align=%d S=%d (%6zu B smem): useful %5.0f GB/s, copied %5.0f GB/s  %s\n", R, rows, align, S,
           smem, gu, gc, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
