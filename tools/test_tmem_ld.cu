// TMEM load semantics on sm_100a (developer check): tcgen05.ld.32x32b.x32 at an unaligned column, and at a
// column window that runs past the 512-column allocation.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void k(int col, int* out) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&base)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = base + (static_cast<uint32_t>(warp * 32) << 16);
  for (int c0 = 0; c0 < 512; c0 += 8) {
    uint32_t v[8];
    for (int j = 0; j < 8; ++j) v[j] = (warp * 32 + lane) * 1000 + c0 + j;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(t + c0), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(t + col) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  int bad = 0;
  for (int j = 0; j < 8; ++j) bad += (col + j < 512 && r[j] != static_cast<uint32_t>((warp * 32 + lane) * 1000 + col + j)) ? 1 : 0;
  atomicAdd(out, bad);
  if (threadIdx.x == 37) out[1] = r[0];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}
int main() {
  int* d;
  cudaMalloc(&d, 8);
  const int cols[] = {0, 5, 13, 250, 503, 508};
  for (int col : cols) {
    cudaMemset(d, 0, 8);
    k<<<1, 128>>>(col, d);
    cudaError_t e = cudaDeviceSynchronize();
    int h[2] = {-1, -1};
    if (e == cudaSuccess) cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("col %d: %s mismatches %d sample %d\n", col, cudaGetErrorString(e), h[0], h[1]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
