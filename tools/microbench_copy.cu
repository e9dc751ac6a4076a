// Developer microbenchmark (not part of the library): achievable global->shared
// bandwidth on this GPU for (a) cp.async.bulk rings of S stages x B bytes per SM,
// (b) plain coalesced 16-byte loads.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
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

__global__ void bulk_ring(const char* src, size_t per_cta, int S, int B, int pieces, int* sink, size_t total,
                          int random) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ uint64_t full[16], empty[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const char* base = src + blockIdx.x * per_cta;
  const int iters = (int)(per_cta / B);
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      int s = i % S;
      wait(&empty[s], ((i / S) & 1) ^ 1);
      arrive_tx(&full[s], B);
      const int pb = B / pieces;
      for (int p = 0; p < pieces; ++p) {
        const char* from = base + (size_t)i * B + p * pb;
        if (random) {  // pseudo-random 128-byte aligned source offsets over the whole buffer
          unsigned long long h = (unsigned long long)(blockIdx.x * 1000003ull + i * 131ull + p) * 0x9E3779B97F4A7C15ull;
          from = src + ((h >> 20) % ((total - pb) / 128)) * 128;
        }
        bulk(su32(sm + s * B + p * pb), from, pb, &full[s]);
      }
    }
  } else if (threadIdx.x == 32) {
    int acc = 0;
    for (int i = 0; i < iters; ++i) {
      int s = i % S;
      wait(&full[s], (i / S) & 1);
      acc += sm[s * B];
      arrive(&empty[s]);
    }
    if (acc == 12345) *sink = acc;
  }
}

// lane-parallel issue: warp 0 issues `pieces` copies per stage, one per lane (pieces <= 32)
__global__ void bulk_ring_lanes(const char* src, size_t per_cta, int S, int B, int pieces, int* sink, size_t span) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ uint64_t full[16], empty[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int iters = (int)(per_cta / B);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    for (int i = 0; i < iters; ++i) {
      int s = i % S;
      wait(&empty[s], ((i / S) & 1) ^ 1);
      if (lane == 0) arrive_tx(&full[s], B);
      __syncwarp();
      const int pb = B / pieces;
      if (lane < pieces) {
        unsigned long long h = (unsigned long long)(blockIdx.x * 1000003ull + i * 131ull + lane) * 0x9E3779B97F4A7C15ull;
        const char* from = src + ((h >> 20) % ((span - pb) / 128)) * 128;
        bulk(su32(sm + s * B + lane * pb), from, pb, &full[s]);
      }
    }
  } else if (threadIdx.x == 32) {
    int acc = 0;
    for (int i = 0; i < iters; ++i) {
      int s = i % S;
      wait(&full[s], (i / S) & 1);
      acc += sm[s * B];
      arrive(&empty[s]);
    }
    if (acc == 12345) *sink = acc;
  }
}

__global__ void ldg_stream(const int4* src, size_t n, int* sink) {
  int4 a = make_int4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int4 v = __ldg(src + i);
    a.x ^= v.x; a.y ^= v.y; a.z ^= v.z; a.w ^= v.w;
  }
  if ((a.x ^ a.y ^ a.z ^ a.w) == 0x7fffffff) *sink = a.x;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)16 << 30;  // 16 GB
  char* src;
  int* sink;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 4);
  cudaMemset(src, 1, total);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // plain loads
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    ldg_stream<<<sms * 8, 256>>>((const int4*)src, total / 16, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("ldg.128 stream          : %.0f GB/s\n", total / ms / 1e6);
  cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int cfgs[][3] = {{2, 16384, 1}, {4, 16384, 1}, {6, 20480, 1}, {8, 16384, 1}, {4, 32768, 1}, {6, 32768, 1},
                   {3, 65536, 1}, {6, 20480, 8}, {6, 20480, 16}, {12, 16384, 1}, {6, 20480, 32}};
  for (int rnd = 0; rnd < 2; ++rnd)
  for (auto& c : cfgs) {
    const int S = c[0], B = c[1], P = c[2];
    if ((size_t)S * B > 200 * 1024) continue;
    for (int ctas_per_sm = 1; ctas_per_sm <= 1; ++ctas_per_sm) {
      const int grid = sms * ctas_per_sm;
      size_t per = (total / grid) / B * B;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        bulk_ring<<<grid, 64, S * B>>>(src, per, S, B, P, sink, total, rnd);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      cudaError_t err = cudaGetLastError();
      printf("bulk ring %s S=%2d B=%6d pieces=%2d : %.0f GB/s  (%s)\n", rnd ? "random" : "stream", S, B, P,
             per * (double)grid / ms / 1e6,
             cudaGetErrorString(err));
    }
  }
  cudaFuncSetAttribute(bulk_ring_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int cfg2[][3] = {{6, 20480, 8}, {6, 20480, 16}, {3, 49152, 6}, {3, 61440, 4}, {2, 98304, 6}, {4, 40960, 4},
                   {4, 40960, 8}, {6, 30720, 12}};
  size_t spans[] = {total, (size_t)192 << 20};
  for (size_t span : spans)
    for (auto& c : cfg2) {
      const int S = c[0], B = c[1], P = c[2];
      const int grid = sms;
      size_t per = ((size_t)4 << 30) / grid / B * B;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        bulk_ring_lanes<<<grid, 64, S * B>>>(src, per, S, B, P, sink, span);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      printf("lanes random span=%5zu MB S=%d B=%6d pieces=%2d (%5d B each): %.0f GB/s (%s)\n", span >> 20, S, B, P,
             B / P, per * (double)grid / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
