// gate.cu — the paper's candidate-generation variants beyond the open sketch scan:
//
//  * BioVSS++ stage 1 (Alg 6 lines 1, 3-9; the inverted index of
//    Alg 4 / Def 9): the query's count Bloom filter C_Q picks its A
//    largest positions P (ties -> lower position, reading R27) and a set passes
//    iff C_i[p] >= M for some p in P.  On the GPU the inverted lists become
//    bit planes: plane p holds one bit per set, (C_i[p] >= M) (a count index) or
//    S_i[p] (a binary index, exact for M = 1 since S = (C > 0)).  The gate of a
//    (query, 32-set word) is then the OR of A plane words; sets that fail it get
//    the key's top bit, so an exact top-T select over the keys returns the
//    first T of F1 by (score, id) and the emission drops everything at or above
//    that bit (|F1| < T gives F2 = F1, as Alg 6 does).
//  * BioVSS Alg 2: the candidate score of a set is the
//    Hamming-Hausdorff distance Haus^H(Q^H, H_j) over the
//    per-vector codes, written as a key row for the same exact top-c select.
//    SIMT: one warp per (query, set), lanes = set vectors, popc over XORed code
//    words; the row minima by redux.sync over the lanes, the column minima per
//    lane.
#include "tc.cuh"

namespace bvss {

// planes[p][w]: bit j = (counter p of set 32w + j) >= M (count sketches) / sketch bit p (binary); chunk-major
// sketches: word w of set i (row-major words) at S[((w / 4) * n + i) * 4 + w % 4]
__global__ void gate_planes_kernel(const uint32_t* __restrict__ S, int64_t n, int m, int kind, int M,
                                   uint32_t* __restrict__ planes, int64_t W) {
  const int64_t total = static_cast<int64_t>(m) * W;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(t / W);
    const int64_t w = t - static_cast<int64_t>(p) * W;
    const int word = kind == BVSS_SKETCH_BINARY ? (p >> 5) : (p >> 2);
    uint32_t bits = 0;
    for (int j = 0; j < 32; ++j) {
      const int64_t i = w * 32 + j;
      if (i >= n) break;
      const uint32_t v = S[((word >> 2) * n + i) * 4 + (word & 3)];
      const bool pass = kind == BVSS_SKETCH_BINARY ? ((v >> (p & 31)) & 1u) != 0u
                                                   : static_cast<int>((v >> (8 * (p & 3))) & 0xFFu) >= M;
      bits |= pass ? (1u << j) : 0u;
    }
    planes[t] = bits;
  }
}

// per query: C_Q = the column sums of its codes (Def 8), then its A largest positions, ties -> lower
// position (reading R27).  One CTA per query.
__global__ void gate_positions_kernel(const uint32_t* __restrict__ qcodes, const int64_t* __restrict__ qoff, int m,
                                      int A, int32_t* __restrict__ pos) {
  extern __shared__ int cnt[];  // [m]
  __shared__ unsigned long long best;
  const int q = blockIdx.x;
  const int R = m / 32;
  for (int p = threadIdx.x; p < m; p += blockDim.x) cnt[p] = 0;
  __syncthreads();
  for (int64_t v = qoff[q]; v < qoff[q + 1]; ++v)
    for (int p = threadIdx.x; p < m; p += blockDim.x) cnt[p] += (qcodes[v * R + (p >> 5)] >> (p & 31)) & 1u;
  __syncthreads();
  for (int a = 0; a < A; ++a) {  // argmax by (count desc, position asc): the key (count << 32) | ~position
    if (threadIdx.x == 0) best = 0ull;
    __syncthreads();
    unsigned long long b = 0ull;
    for (int p = threadIdx.x; p < m; p += blockDim.x)
      if (cnt[p] >= 0) {
        const unsigned long long key = (static_cast<unsigned long long>(cnt[p] + 1) << 32) | (0xFFFFFFFFu - p);
        b = key > b ? key : b;
      }
    atomicMax(&best, b);
    __syncthreads();
    const int p = static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(best & 0xFFFFFFFFull));
    if (threadIdx.x == 0) {
      pos[static_cast<int64_t>(q) * A + a] = p;
      cnt[p] = -1;  // taken
    }
    __syncthreads();
  }
}

// keys[q][i] |= high where set i fails the gate of query q (no p in P_q with C_i[p] >= M)
template <typename K>
__global__ void gate_keys_kernel(K* __restrict__ keys, int64_t key_stride, int64_t n, int nq,
                                 const int32_t* __restrict__ pos, int A, const uint32_t* __restrict__ planes,
                                 int64_t W, K high) {
  const int64_t total = static_cast<int64_t>(nq) * W;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int q = static_cast<int>(t / W);
    const int64_t w = t - static_cast<int64_t>(q) * W;
    uint32_t g = 0;
    for (int a = 0; a < A; ++a) g |= planes[static_cast<int64_t>(pos[static_cast<int64_t>(q) * A + a]) * W + w];
    K* row = keys + static_cast<int64_t>(q) * key_stride;
    for (int j = 0; j < 32; ++j) {
      const int64_t i = w * 32 + j;
      if (i >= n) break;
      if (((g >> j) & 1u) == 0u) row[i] = static_cast<K>(row[i] | high);
    }
  }
}

// Alg 2: keys[q][i] = Haus^H(Q^H_q, H_i) = max(max_q min_v ham, max_v min_q ham), ham = popc(h_q XOR h_v).
// Grid (set blocks, queries); one warp per set at a time; the query's codes in shared memory.
__global__ void __launch_bounds__(256) alg2_keys_kernel(const uint32_t* __restrict__ qcodes,
                                                        const int64_t* __restrict__ qoff, const uint32_t* __restrict__ codes,
                                                        const int64_t* __restrict__ off, int64_t n, int R,
                                                        uint16_t* __restrict__ keys, int64_t key_stride,
                                                        int max_mq) {
  extern __shared__ uint32_t qs[];  // [m_q][R] query codes, then [8 warps][max_mq] row minima
  const int q = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q0 = qoff[q];
  const int mq = static_cast<int>(qoff[q + 1] - q0);
  for (int t = threadIdx.x; t < mq * R; t += blockDim.x) qs[t] = qcodes[q0 * R + t];
  uint32_t* rowmin = qs + static_cast<size_t>(max_mq) * R + static_cast<size_t>(warp) * max_mq;
  __syncthreads();
  const int64_t per_block = (n + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = blockIdx.x * per_block, i1 = min(n, i0 + per_block);
  for (int64_t i = i0 + warp; i < i1; i += 8) {
    const int64_t v0 = off[i];
    const int mv = static_cast<int>(off[i + 1] - v0);
    for (int a = lane; a < mq; a += 32) rowmin[a] = 0xFFFFFFFFu;
    __syncwarp();
    uint32_t hv = 0;  // max over v of min over q
    for (int b = 0; b < mv; b += 32) {
      const bool vv = b + lane < mv;
      const uint32_t* vc = codes + (v0 + (vv ? b + lane : 0)) * R;
      uint32_t colmin = 0xFFFFFFFFu;
      for (int a = 0; a < mq; ++a) {
        uint32_t h = 0;
        for (int w = 0; w < R; ++w) h += __popc(qs[a * R + w] ^ __ldg(vc + w));
        colmin = min(colmin, h);
        const uint32_t rm = __reduce_min_sync(0xffffffffu, vv ? h : 0xFFFFFFFFu);
        if (lane == 0) rowmin[a] = min(rowmin[a], rm);
      }
      hv = max(hv, vv ? colmin : 0u);
    }
    __syncwarp();
    uint32_t hq = 0;
    for (int a = lane; a < mq; a += 32) hq = max(hq, rowmin[a]);
    hq = __reduce_max_sync(0xffffffffu, hq);
    hv = __reduce_max_sync(0xffffffffu, hv);
    if (lane == 0) keys[static_cast<int64_t>(q) * key_stride + i] = static_cast<uint16_t>(max(hq, hv));
    __syncwarp();
  }
}

int launch_gate_planes(const void* S, int64_t n, int m, int kind, int M, uint32_t* planes, int64_t W, int num_sms,
                       cudaStream_t st) {
  gate_planes_kernel<<<num_sms * 8, 256, 0, st>>>(static_cast<const uint32_t*>(S), n, m, kind, M, planes, W);
  return post_launch("gate_planes_kernel", st);
}

int launch_gate_positions(const uint32_t* qcodes, const int64_t* qoff, int nq, int m, int A, int32_t* pos,
                          cudaStream_t st) {
  if (nq <= 0) return BVSS_OK;
  gate_positions_kernel<<<nq, 256, static_cast<size_t>(m) * sizeof(int), st>>>(qcodes, qoff, m, A, pos);
  return post_launch("gate_positions_kernel", st);
}

int launch_gate_keys(int key_size, void* keys, int64_t key_stride, int64_t n, int nq, const int32_t* pos, int A,
                     const uint32_t* planes, int64_t W, int num_sms, cudaStream_t st) {
  if (nq <= 0) return BVSS_OK;
  if (key_size == 2)
    gate_keys_kernel<uint16_t><<<num_sms * 8, 256, 0, st>>>(static_cast<uint16_t*>(keys), key_stride, n, nq, pos, A,
                                                             planes, W, static_cast<uint16_t>(0x8000u));
  else
    gate_keys_kernel<uint32_t><<<num_sms * 8, 256, 0, st>>>(static_cast<uint32_t*>(keys), key_stride, n, nq, pos, A,
                                                             planes, W, 0x80000000u);
  return post_launch("gate_keys_kernel", st);
}

int launch_alg2_keys(const uint32_t* qcodes, const int64_t* qoff, int nq, int max_mq, const uint32_t* codes,
                     const int64_t* off, int64_t n, int m, uint16_t* keys, int64_t key_stride, int num_sms,
                     cudaStream_t st) {
  if (nq <= 0) return BVSS_OK;
  const int R = m / 32;
  const size_t smem = (static_cast<size_t>(max_mq) * R + 8 * static_cast<size_t>(max_mq)) * 4;
  if (smem > 200 * 1024) BVSS_FAIL(BVSS_EUNSUPPORTED, "Alg 2 scan: query set too large for shared memory");
  BVSS_CUDA(cudaFuncSetAttribute(alg2_keys_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int bx = static_cast<int>((static_cast<int64_t>(num_sms) * 8 + nq - 1) / nq);
  if (bx < 1) bx = 1;
  if (bx > 4096) bx = 4096;
  const dim3 grid(static_cast<unsigned>(bx), static_cast<unsigned>(nq));
  alg2_keys_kernel<<<grid, 256, smem, st>>>(qcodes, qoff, codes, off, n, R, keys, key_stride, max_mq);
  return post_launch("alg2_keys_kernel", st);
}

}  // namespace bvss
