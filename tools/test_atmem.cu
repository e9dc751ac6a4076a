// Developer check (not part of the library): the A-operand-in-TMEM form of the refine Gram.
// The query rows (SW128 K-major, 2 K-chunks per 8-row group: SBO = 2 KB, as in refine.cu) are
// copied smem -> TMEM by tcgen05.cp (32x128b.warpx4 / 64x128b.warpx2::02_13 / 128x128b,
// replicating them over the 4 TMEM lane quarters), then tcgen05.mma kind::f16 with A in TMEM
// and B (160 candidate rows, same layout) in smem; D at TMEM column 160, A at 320.  D is
// compared on the host with a double-precision Gram of the same fp16 values.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../paper_2412_03301_b200/csrc test_atmem.cu -o test_atmem
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc.cuh"

using namespace bvss;

constexpr int K = 384, KS = 3, KCS = 2, NB = 160;

__device__ __forceinline__ uint64_t desc_sbo(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

__global__ void kern(const uint8_t* gA, int a_rows, const uint8_t* gB, float* out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  const int a_bytes = a_rows * K * 2, b_bytes = NB * K * 2;
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
  const uint32_t tm = tbase, tD = tm + 160, tA = tm + 320;
  if (threadIdx.x == 0) {
    const uint32_t sA = smem_u32(sm), sB = sA + a_bytes;
    const uint32_t ssA = a_rows / 8 * KCS * 1024, ssB = NB / 8 * KCS * 1024;
    for (int ks = 0; ks < KS; ++ks)
      for (int kc = 0; kc < KCS; ++kc)
        for (int j = 0; j < 8; ++j) {
          const uint32_t col = tA + (ks * KCS + kc) * 32 + j * 4;
          const uint64_t d = desc_sbo(sA + ks * ssA + kc * 1024 + j * 16, KCS * 1024);
          if (mode == 32)
            asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(col), "l"(d) : "memory");
          else if (mode == 64)
            asm volatile("tcgen05.cp.cta_group::1.64x128b.warpx2::02_13 [%0], %1;" ::"r"(col), "l"(d) : "memory");
          else
            asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(col), "l"(d) : "memory");
        }
    const uint32_t idesc = tc::idesc_f16_f32(128, NB);
    for (int ks = 0; ks < KS; ++ks)
      for (int kc = 0; kc < KCS; ++kc)
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t a_col = tA + (ks * KCS + kc) * 32 + kk * 8;
          const uint64_t bd = desc_sbo(sB + ks * ssB + kc * 1024 + kk * 32, KCS * 1024);
          const uint32_t acc = (ks | kc | kk) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tD),
              "r"(a_col), "l"(bd), "r"(idesc), "r"(acc)
              : "memory");
        }
    tc::umma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  for (int c = 0; c < NB; c += 16) {
    uint32_t r[16];
    tc::tmem_ld16(tD + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
    tc::tmem_ld_wait();
    for (int i = 0; i < 16; ++i) out[(warp * 32 + lane) * NB + c + i] = __uint_as_float(r[i]);
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0) tc::tmem_dealloc(tm, 512);
}

// host: element (r, k) of a [rows][K] matrix -> byte offset in the pre-swizzled layout
static size_t off(int rows, int r, int k) {
  const int ks = k / 128, kc = (k % 128) / 64, e = k % 64, u = e / 8, w = e % 8;
  return static_cast<size_t>(ks) * (rows / 8) * KCS * 1024 + (r / 8) * KCS * 1024 + kc * 1024 + (r % 8) * 128 +
         ((u ^ (r % 8)) * 16) + w * 2;
}

int main() {
  int bad_total = 0;
  for (int mode : {32, 64, 128}) {
    const int ar = mode;
    std::vector<float> A(ar * K), B(NB * K);
    srand(1234 + mode);
    for (auto& x : A) x = __half2float(__float2half((rand() % 2001 - 1000) / 1000.0f));
    for (auto& x : B) x = __half2float(__float2half((rand() % 2001 - 1000) / 1000.0f));
    std::vector<uint8_t> hA(ar * K * 2), hB(NB * K * 2);
    for (int r = 0; r < ar; ++r)
      for (int k = 0; k < K; ++k) *reinterpret_cast<__half*>(&hA[off(ar, r, k)]) = __float2half(A[r * K + k]);
    for (int r = 0; r < NB; ++r)
      for (int k = 0; k < K; ++k) *reinterpret_cast<__half*>(&hB[off(NB, r, k)]) = __float2half(B[r * K + k]);
    uint8_t *dA, *dB;
    float* dO;
    cudaMalloc(&dA, hA.size());
    cudaMalloc(&dB, hB.size());
    cudaMalloc(&dO, 128 * NB * 4);
    cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
    kern<<<1, 128, (ar + NB) * K * 2 + 1024>>>(dA, ar, dB, dO, mode);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    std::vector<float> O(128 * NB);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    double maxerr = 0;
    for (int l = 0; l < 128; ++l) {
      const int row = mode == 32 ? l % 32 : (mode == 64 ? l % 64 : l);
      for (int n = 0; n < NB; ++n) {
        double g = 0;
        for (int k = 0; k < K; ++k) g += static_cast<double>(A[row * K + k]) * B[n * K + k];
        const double err = fabs(g - O[l * NB + n]);
        maxerr = fmax(maxerr, err);
        if (err > 1e-3 + 1e-4 * fabs(g)) {
          if (bad < 3) printf("  mode %d lane %d col %d: got %f want %f\n", mode, l, n, O[l * NB + n], g);
          ++bad;
        }
      }
    }
    printf("mode %3d: %s, mismatches %d, max |err| %.2e\n", mode, cudaGetErrorString(e), bad, maxerr);
    bad_total += bad + (e != cudaSuccess);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dO);
  }
  printf(bad_total ? "FAIL\n" : "PASS\n");
  return bad_total ? 1 : 0;
}
