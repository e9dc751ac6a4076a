// Developer check (not part of the library): where does tcgen05.mma.ws (weight-stationary) with a small
// M put the accumulator in TMEM?  (an M = 32 A operand without replicas would free a third
// of each refine stage if the N columns spread over the four TMEM lane quarters.)
// A[i][k] = (k == 0 ? i : k == 1 ? 1 : 0), B[j][k] = (k == 0 ? 1 : k == 1 ? 256 j : 0)  =>  D[i][j] = i + 256 j.
// The kernel dumps TMEM lanes 0..127 x columns 0..255 and the host decodes every non-zero value.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../paper_2412_03301_b200/csrc test_ws.cu -o test_ws
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "tc.cuh"

using namespace bvss;

constexpr int K = 64;  // one SW128 K-chunk

__device__ __forceinline__ uint64_t desc_sbo(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

__global__ void kern(const uint8_t* gA, int M, const uint8_t* gB, int N, float* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  const int a_bytes = 128 * K * 2, b_bytes = N * K * 2;  // A buffer sized for 128 rows (rows >= M are zero)
  for (int i = threadIdx.x; i < a_bytes / 16; i += blockDim.x)
    reinterpret_cast<int4*>(sm)[i] = reinterpret_cast<const int4*>(gA)[i];
  for (int i = threadIdx.x; i < b_bytes / 16; i += blockDim.x)
    reinterpret_cast<int4*>(sm + a_bytes)[i] = reinterpret_cast<const int4*>(gB)[i];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tm = tbase;
  // zero the dump region first (so unwritten cells read 0)
  for (int c = 0; c < 256; c += 1) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tm + (static_cast<uint32_t>(warp * 32) << 16) + c),
                 "r"(0u)
                 : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (threadIdx.x == 0) {
    const uint32_t sA = smem_u32(sm), sB = sA + a_bytes;
    const uint32_t idesc = tc::idesc_f16_f32(M, N);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t ad = desc_sbo(sA + kk * 32, 1024), bd = desc_sbo(sB + kk * 32, 1024);
      const uint32_t acc = kk ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.ws.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
          : "memory");
    }
    tc::umma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  for (int c = 0; c < 256; c += 16) {
    uint32_t r[16];
    tc::tmem_ld16(tm + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
    tc::tmem_ld_wait();
    for (int i = 0; i < 16; ++i) out[(warp * 32 + lane) * 256 + c + i] = __uint_as_float(r[i]);
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0) tc::tmem_dealloc(tm, 512);
}

static size_t off(int r, int k) {  // SW128 K-major, one K-chunk: 8-row groups of 1 KB
  const int u = k / 8, w = k % 8;
  return static_cast<size_t>(r / 8) * 1024 + (r % 8) * 128 + ((u ^ (r % 8)) * 16) + w * 2;
}

int main() {
  const int shapes[][2] = {{32, 256}, {64, 256}, {32, 128}, {128, 256}};
  for (auto& sh : shapes) {
    const int M = sh[0], N = sh[1];
    std::vector<uint8_t> hA(128 * K * 2, 0), hB(N * K * 2, 0);
    for (int i = 0; i < M; ++i) {
      *reinterpret_cast<__half*>(&hA[off(i, 0)]) = __float2half(static_cast<float>(i));
      *reinterpret_cast<__half*>(&hA[off(i, 1)]) = __float2half(1.0f);
    }
    for (int j = 0; j < N; ++j) {
      *reinterpret_cast<__half*>(&hB[off(j, 0)]) = __float2half(1.0f);
      *reinterpret_cast<__half*>(&hB[off(j, 1)]) = __float2half(256.0f * j);
    }
    uint8_t *dA, *dB;
    float* dO;
    cudaMalloc(&dA, hA.size());
    cudaMalloc(&dB, hB.size());
    cudaMalloc(&dO, 128 * 256 * 4);
    cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    kern<<<1, 128, 128 * K * 2 + N * K * 2 + 1024>>>(dA, M, dB, N, dO);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    std::vector<float> O(128 * 256);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    printf("M=%d N=%d: %s\n", M, N, cudaGetErrorString(e));
    // per lane quarter: which rows i and column range j land there
    int hits = 0;
    for (int q = 0; q < 4; ++q) {
      int imin = 1 << 30, imax = -1, jmin = 1 << 30, jmax = -1, cmin = 1 << 30, cmax = -1, cnt = 0;
      for (int l = 32 * q; l < 32 * q + 32; ++l)
        for (int c = 0; c < 256; ++c) {
          const float v = O[l * 256 + c];
          const int iv = static_cast<int>(v);
          if (v == 0.0f || static_cast<float>(iv) != v) continue;
          const int i = iv % 256, j = iv / 256;
          ++cnt;
          imin = i < imin ? i : imin; imax = i > imax ? i : imax;
          jmin = j < jmin ? j : jmin; jmax = j > jmax ? j : jmax;
          cmin = c < cmin ? c : cmin; cmax = c > cmax ? c : cmax;
        }
      hits += cnt;
      if (cnt)
        printf("  lanes %3d-%3d: %5d values, rows i %3d..%3d, cols j %3d..%3d at TMEM columns %3d..%3d\n", 32 * q,
               32 * q + 31, cnt, imin, imax, jmin, jmax, cmin, cmax);
    }
    // spot-check: the lane/column of a few (i, j)
    for (int l = 0; l < 128; l += 37)
      printf("  lane %3d col 0..3: %g %g %g %g\n", l, O[l * 256], O[l * 256 + 1], O[l * 256 + 2], O[l * 256 + 3]);
    printf("  total nonzero %d (expect %d minus the i=0,j=0 cell)\n", hits, M * N);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dO);
  }
  return 0;
}
