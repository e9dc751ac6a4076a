// Developer microbenchmark (not part of the library): cycles per tcgen05.mma
// (kind::f16, cta_group::1, M=128, K=16, SS operands, SW128 K-major) as a function
// of N, issued back to back by one thread from smem-resident operands.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../paper_2412_03301_b200/csrc
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc.cuh"

using namespace bvss;

__global__ void umma_loop(int N, int iters, int nacc, int m, unsigned long long* out, int ts) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) base[i] = 0;  // A: 128 x 128B (16 KB), B: up to 256 x 128B
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  if (warp == 0 && (ts >= 2 || lane == 0)) {  // ts >= 2: the whole warp runs the loop, elect.sync issues
    const uint32_t a = smem_u32(base), b = a + 16384;
    const uint32_t idesc = tc::idesc_f16_f32(m, N);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t d = tbase + ((it * 4 + kk) % nacc) * N;
        if (ts >= 2) {  // convergent warp, elect.sync inside the asm; 2 = SS, 3 = TS
          const uint32_t en = (it | kk) ? 1u : 0u;
          if (ts == 2)
            asm volatile(
                "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                "l"(tc::sw128_desc(a + kk * 32)), "l"(tc::sw128_desc(b + kk * 32)), "r"(idesc), "r"(en)
                : "memory");
          else
            asm volatile(
                "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                "r"(tbase + 480 + kk * 8), "l"(tc::sw128_desc(b + kk * 32)), "r"(idesc), "r"(en)
                : "memory");
        } else if (ts) {  // A in TMEM (columns 480 + 8 kk)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
              "r"(tbase + 480 + kk * 8), "l"(tc::sw128_desc(b + kk * 32)), "r"(idesc), "r"((it | kk) ? 1u : 0u)
              : "memory");
        } else {
          tc::umma_bf16(d, tc::sw128_desc(a + kk * 32), tc::sw128_desc(b + kk * 32), idesc, (it | kk) ? 1u : 0u);
        }
      }
    }
    if (ts < 2 || lane == 0) tc::umma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  cudaFuncSetAttribute(umma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 2000;
  int Ns[] = {64, 128, 256};
  for (int ts : {0, 2, 3})
  for (int m : {128})
    for (int nacc : {1, 2})
      for (int N : Ns) {
        if (N * nacc > 480) continue;
        if (m == 128 && N % 16) continue;
        for (int grid : {148}) {
          printf("%s%s ", ts & 1 ? "TS" : "SS", ts >= 2 ? "-warp" : "");
          umma_loop<<<grid, 128, 100 * 1024>>>(N, iters, nacc, m, d, ts);
          cudaError_t e = cudaDeviceSynchronize();
          unsigned long long h = 0;
          cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
          const double per = (double)h / (iters * 4);
          printf("M=%3d N=%3d acc=%d grid=%3d: %.1f cycles/UMMA  (%.0f MAC/clk/SM)  %s\n", m, N, nacc, grid, per,
                 m * N * 16 / per, cudaGetErrorString(e));
        }
      }
  return 0;
}
