// Developer microbenchmark (not part of the library): throughput and a value
// check of the two candidate tensor-core forms of the filter scan,
//   kind::i8   (u8 x u8 -> s32, K = 32 bytes per instruction) and
//   kind::mxf4 (e2m1 x e2m1 -> f32, ue8m0 block scales = 1.0, K = 64 elements = 32 bytes),
// M = 128, N = 256 (or 240), no-swizzle K-major operands, issued back to back by one thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../paper_2412_03301_b200/csrc microbench_scan_mma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc.cuh"

using namespace bvss;

__device__ __forceinline__ uint64_t kdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  return d;
}

// mode 0: i8, mode 1: mxf4
__global__ void bench(int mode, int N, int iters, unsigned long long* out, float* val) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // A: 2 K units x 128 rows x 16 B; B: 2 units x 256 rows x 16 B.  Fill: i8 -> 1 everywhere; mxf4 -> 0x22 (1.0, 1.0)
  const uint8_t fill = mode == 0 ? 1 : 0x22;
  for (int i = threadIdx.x; i < 2 * 128 * 16 + 2 * 256 * 16; i += blockDim.x) base[i] = fill;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tm = tbase;
  // scale factors (mxf4): columns [480, 512) of every lane = 0x7F (ue8m0 1.0)
  if (mode == 1) {
    const uint32_t taddr = tm + (static_cast<uint32_t>(warp * 32) << 16) + 480;
    for (int c = 0; c < 32; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr + c), "r"(0x7F7F7F7Fu) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0 && lane == 0) {
    const uint32_t a = smem_u32(base), b = a + 2 * 128 * 16;
    const uint64_t ad = kdesc(a, 128 * 16, 128), bd = kdesc(b, 256 * 16, 128);
    uint32_t idesc;
    if (mode == 0) idesc = (2u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (8u << 24);
    else idesc = (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (1u << 23) | (8u << 24);
    const uint32_t sfa = tm + 480, sfb = tm + 496;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tm + (it & 1) * 240;
      const uint32_t acc = it >= 2 ? 1u : 0u;
      if (mode == 0) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
      }
    }
    tc::umma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = static_cast<unsigned long long>(t1 - t0);
  }
  __syncthreads();
  tc::fence_after_sync();
  // read back D[lane row][col 0] of accumulator 0 (it = 0, 2, 4, ... accumulate: (iters/2) x K)
  if (warp < 4 && blockIdx.x == 0) {
    uint32_t r[16];
    tc::tmem_ld16(tm + (static_cast<uint32_t>(warp * 32) << 16), r);
    tc::tmem_ld_wait();
    if (lane == 5) val[warp] = mode == 0 ? static_cast<float>(static_cast<int32_t>(r[3])) : __uint_as_float(r[3]);
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tm, 512);
}

int main() {
  unsigned long long* d;
  float* v;
  cudaMalloc(&d, 8);
  cudaMalloc(&v, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 4000;
  for (int mode = 0; mode < 2; ++mode)
    for (int N : {240, 256}) {
      if (mode == 1 && N == 256) continue;  // accumulators 2 x 240 + scale columns
      for (int grid : {1, 148}) {
        bench<<<grid, 128, 64 * 1024>>>(mode, N, iters, d, v);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h = 0;
        float hv[4] = {0, 0, 0, 0};
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(hv, v, 16, cudaMemcpyDeviceToHost);
        const double per = static_cast<double>(h) / iters;
        const double kel = mode == 0 ? 32 : 64;
        printf("%s N=%d grid=%3d: %.1f cycles/MMA (%.0f MAC/clk/SM); D[5][3] = %.0f %.0f %.0f %.0f (expect %.0f)  %s\n",
               mode == 0 ? "i8  " : "mxf4", N, grid, per, 128.0 * N * kel / per, hv[0], hv[1], hv[2], hv[3],
               kel * (iters / 2), cudaGetErrorString(e));
      }
    }
  return 0;
}
