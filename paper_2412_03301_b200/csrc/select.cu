// select.cu — K4: exact top-T candidate selection (Alg 6 lines 10-18).
//
// The paper keeps a T-capacity max-heap over the filter scores.  Here the T
// smallest (score, id) pairs per query are found exactly by an MSB-first radix
// select over the score keys (11-bit digits, one histogram round per digit),
// then emitted in ascending id order by an order-preserving block compaction
// that takes every key below the threshold tau and the lowest-id keys equal to
// tau up to the quota (readings R3/R4: one budget T, ties -> lower id).
//
// Each round is split into hist (local) and resolve (global) kernels so that the
// sharded protocol can all-reduce the histograms in between; on
// one GPU the local histogram is the global one.  One CTA per query streams that
// query's key row with 16-byte loads.
#include "common.cuh"

namespace bvss {

struct SelectState {  // device arrays, one entry per query
  uint32_t* prefix;   // resolved high bits of tau
  int64_t* below;     // # keys (global) strictly below the current range
  int64_t* teff;      // min(T, n_total)
  int64_t* eq;        // # keys (global) equal to tau, after the last round
  int64_t* quota;     // # keys equal to tau this rank emits
  int32_t* digit;     // chosen digit of the last resolved round
};

template <typename K>
struct KeyVec;
template <>
struct KeyVec<uint16_t> {
  static constexpr int kPer = 8;
};
template <>
struct KeyVec<uint32_t> {
  static constexpr int kPer = 4;
};

template <typename K>
__device__ __forceinline__ void load_keys(const K* row, int64_t base, int64_t n, K (&k)[8]) {
  // 8 consecutive keys starting at base (16B aligned); out-of-range -> max
  if (base + 8 <= n) {
    if (sizeof(K) == 2) {
      const uint4 v = *reinterpret_cast<const uint4*>(row + base);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        k[2 * i] = static_cast<K>(w[i] & 0xFFFFu);
        k[2 * i + 1] = static_cast<K>(w[i] >> 16);
      }
    } else {
      const uint4 v0 = *reinterpret_cast<const uint4*>(row + base);
      const uint4 v1 = *reinterpret_cast<const uint4*>(row + base + 4);
      k[0] = v0.x; k[1] = v0.y; k[2] = v0.z; k[3] = v0.w;
      k[4] = v1.x; k[5] = v1.y; k[6] = v1.z; k[7] = v1.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) k[i] = (base + i < n) ? row[base + i] : static_cast<K>(~static_cast<K>(0));
  }
}

// ------------------------------------------------------------- histogram --
template <typename K>
__global__ void __launch_bounds__(256) select_hist_kernel(const K* __restrict__ keys, int64_t key_stride, int64_t n,
                                                          SelectState st, int hi, int shift, int width,
                                                          int32_t* __restrict__ hist_out /*[nq][2048]*/) {
  extern __shared__ uint32_t wh[];  // [8 warps][nbins]
  const int q = blockIdx.x;
  const int warp = threadIdx.x >> 5;
  const int nbins = 1 << width;
  for (int i = threadIdx.x; i < 8 * nbins; i += blockDim.x) wh[i] = 0u;
  __syncthreads();
  const uint32_t prefix = st.prefix[q];
  const K* row = keys + static_cast<int64_t>(q) * key_stride;
  uint32_t* myh = wh + warp * nbins;
  const uint32_t mask = static_cast<uint32_t>(nbins) - 1u;
  for (int64_t base = static_cast<int64_t>(threadIdx.x) * 8; base < n; base += static_cast<int64_t>(blockDim.x) * 8) {
    K k[8];
    load_keys<K>(row, base, n, k);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t kk = static_cast<uint32_t>(k[i]);
      const bool in = (base + i < n) && ((hi >= 32) ? true : ((kk >> hi) == prefix));
      if (in) atomicAdd(&myh[(kk >> shift) & mask], 1u);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) {
    uint32_t s = 0;
    if (b < nbins) {
#pragma unroll
      for (int w = 0; w < 8; ++w) s += wh[w * nbins + b];
    }
    hist_out[static_cast<int64_t>(q) * kHistBins + b] = static_cast<int32_t>(s);
  }
}

// --------------------------------------------------------------- resolve --
// One warp per query: find the digit where the cumulative (global) count
// reaches need = teff - below.
__global__ void select_resolve_kernel(const int32_t* __restrict__ hist, SelectState st, int nq, int width, int last) {
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  const int64_t need = st.teff[q] - st.below[q];
  const int32_t* h = hist + static_cast<int64_t>(q) * kHistBins;
  const int nbins = 1 << width;
  int64_t run = 0;
  int chosen = -1;
  int64_t before = 0;
  for (int b0 = 0; b0 < nbins && chosen < 0; b0 += 32) {
    const int b = b0 + lane;
    int64_t v = (b < nbins) ? h[b] : 0;
    int64_t inc = v;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, (b < nbins) && (run + inc >= need));
    if (hit) {
      const int src = __ffs(hit) - 1;
      chosen = b0 + src;
      before = run + __shfl_sync(0xffffffffu, inc - v, src);
    }
    run += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) {
    if (chosen < 0) chosen = nbins - 1;  // unreachable when need <= keys in range
    st.prefix[q] = (st.prefix[q] << width) | static_cast<uint32_t>(chosen);
    st.below[q] += before;
    st.digit[q] = chosen;
    if (last) {
      st.eq[q] = h[chosen];
      st.quota[q] = need - before;  // single shard: all remaining slots go to the ties
    }
  }
}

// Sharded: this rank's quota of ties from the all-gathered local tie counts.
__global__ void select_quota_kernel(SelectState st, const int64_t* __restrict__ all_eq /*[P][nq]*/, int nq, int world,
                                    int rank) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  int64_t left = st.teff[q] - st.below[q];
  for (int r = 0; r < rank; ++r) left -= all_eq[static_cast<int64_t>(r) * nq + q];
  const int64_t mine = all_eq[static_cast<int64_t>(rank) * nq + q];
  st.quota[q] = left < 0 ? 0 : (left > mine ? mine : left);
}

// local count of keys equal to tau (from the rank's last-round local histogram)
__global__ void select_tiecount_kernel(const int32_t* __restrict__ local_hist, SelectState st, int nq,
                                       int64_t* __restrict__ eq_out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  eq_out[q] = local_hist[static_cast<int64_t>(q) * kHistBins + st.digit[q]];
}

// ------------------------------------------------------------------ emit --
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* smem_warp /*[8]*/, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) smem_warp[warp] = inc;
  __syncthreads();
  uint32_t wpre = 0, tot = 0;
  const int nw = blockDim.x >> 5;
  for (int w = 0; w < nw; ++w) {
    const uint32_t x = smem_warp[w];
    if (w < warp) wpre += x;
    tot += x;
  }
  __syncthreads();
  total = tot;
  return wpre + inc - v;
}

template <typename K>
__global__ void __launch_bounds__(256) select_emit_kernel(const K* __restrict__ keys, int64_t key_stride, int64_t n,
                                                          SelectState st, int T, int64_t id_base,
                                                          int32_t* __restrict__ cand, int32_t* __restrict__ score,
                                                          int32_t* __restrict__ count, uint32_t key_limit) {
  __shared__ uint32_t sw[8];
  const int q = blockIdx.x;
  const uint32_t tau = st.prefix[q];
  const int64_t quota = st.quota[q];
  const K* row = keys + static_cast<int64_t>(q) * key_stride;
  int32_t* crow = cand + static_cast<int64_t>(q) * T;
  int32_t* srow = score ? score + static_cast<int64_t>(q) * T : nullptr;
  int64_t taken = 0, eq_seen = 0;
  for (int64_t tile = 0; tile < n && taken < T; tile += static_cast<int64_t>(blockDim.x) * 8) {
    const int64_t base = tile + static_cast<int64_t>(threadIdx.x) * 8;
    K k[8];
    uint32_t nlt = 0, neq = 0;
    if (base < n) {
      load_keys<K>(row, base, n, k);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t kk = static_cast<uint32_t>(k[i]);
        const bool valid = base + i < n;
        nlt += (valid && kk < tau && kk < key_limit) ? 1u : 0u;  // key_limit: keys at or above it (the stage-1
        neq += (valid && kk == tau && kk < key_limit) ? 1u : 0u; // gate's rejects, gate.cu) are never taken
      }
    }
    uint32_t total;
    const uint32_t ex = block_exclusive_scan(nlt | (neq << 16), sw, total);
    const int64_t lt_pre = ex & 0xFFFFu, eq_pre = ex >> 16;
    int64_t eq_room = quota - eq_seen;  // ties still to take, in id order
    if (eq_room < 0) eq_room = 0;
    int64_t pos = taken + lt_pre + (eq_pre < eq_room ? eq_pre : eq_room);
    int64_t my_eq = eq_seen + eq_pre;
    if (base < n) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t kk = static_cast<uint32_t>(k[i]);
        if (base + i >= n) break;
        bool take = false;
        if (kk >= key_limit) take = false;
        else if (kk < tau) take = true;
        else if (kk == tau) { take = my_eq < quota; ++my_eq; }
        if (take && pos < T) {
          crow[pos] = static_cast<int32_t>(id_base + base + i);
          if (srow) srow[pos] = static_cast<int32_t>(kk);
          ++pos;
        }
      }
    }
    const int64_t tlt = total & 0xFFFFu, teq = total >> 16;
    taken += tlt + (teq < eq_room ? teq : eq_room);
    eq_seen += teq;
  }
  if (taken > T) taken = T;
  for (int64_t i = taken + threadIdx.x; i < T; i += blockDim.x) {
    crow[i] = -1;
    if (srow) srow[i] = -1;
  }
  if (threadIdx.x == 0 && count) count[q] = static_cast<int32_t>(taken);
}

// The same selection as select_emit_kernel, written as a bitmap (bit i of word i/32 of the query's row =
// set i is one of its top-T candidates): the candidate restriction of the dense refine (dense.cu) at large T,
// where [nq][T] id lists would not fit.  The bitmap must be zero on entry.
template <typename K>
__global__ void __launch_bounds__(256) select_bitmap_kernel(const K* __restrict__ keys, int64_t key_stride, int64_t n,
                                                            SelectState st, int T, uint32_t* __restrict__ bitmap,
                                                            int64_t words, uint32_t key_limit) {
  __shared__ uint32_t sw[8];
  const int q = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const uint32_t tau = st.prefix[q];
  const int64_t quota = st.quota[q];
  const K* row = keys + static_cast<int64_t>(q) * key_stride;
  uint32_t* brow = bitmap + static_cast<int64_t>(q) * words;
  int64_t taken = 0, eq_seen = 0;
  for (int64_t tile = 0; tile < n && taken < T; tile += static_cast<int64_t>(blockDim.x) * 8) {
    const int64_t base = tile + static_cast<int64_t>(threadIdx.x) * 8;
    K k[8];
    uint32_t nlt = 0, neq = 0;
    if (base < n) {
      load_keys<K>(row, base, n, k);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t kk = static_cast<uint32_t>(k[i]);
        const bool valid = base + i < n;
        nlt += (valid && kk < tau && kk < key_limit) ? 1u : 0u;  // key_limit: keys at or above it (the stage-1
        neq += (valid && kk == tau && kk < key_limit) ? 1u : 0u; // gate's rejects, gate.cu) are never taken
      }
    }
    uint32_t total;
    const uint32_t ex = block_exclusive_scan(nlt | (neq << 16), sw, total);
    const int64_t eq_pre = ex >> 16;
    int64_t eq_room = quota - eq_seen;
    if (eq_room < 0) eq_room = 0;
    int64_t my_eq = eq_seen + eq_pre;
    uint32_t bits = 0;
    if (base < n) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t kk = static_cast<uint32_t>(k[i]);
        if (base + i >= n) break;
        bool take = false;
        if (kk >= key_limit) take = false;
        else if (kk < tau) take = true;
        else if (kk == tau) { take = my_eq < quota; ++my_eq; }
        if (take) bits |= 1u << i;
      }
    }
    uint32_t w = bits << (8 * (lane & 3));  // 4 threads x 8 ids = one 32-id word
    w |= __shfl_xor_sync(0xffffffffu, w, 1);
    w |= __shfl_xor_sync(0xffffffffu, w, 2);
    if ((lane & 3) == 0 && base < n) brow[base >> 5] = w;
    const int64_t tlt = total & 0xFFFFu, teq = total >> 16;
    taken += tlt + (teq < eq_room ? teq : eq_room);
    eq_seen += teq;
  }
}

// --------------------------------------------------------------- drivers --
__global__ void select_init_kernel(SelectState st, int nq, int64_t teff) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  st.prefix[q] = 0u;
  st.below[q] = 0;
  st.teff[q] = teff;
  st.eq[q] = 0;
  st.quota[q] = 0;
  st.digit[q] = 0;
}

int key_bits_for(int kind, int m) {
  uint64_t maxkey = kind == BVSS_SKETCH_BINARY ? static_cast<uint64_t>(m) : static_cast<uint64_t>(m) * 255u * 255u;
  int b = 1;
  while ((maxkey >> b) != 0) ++b;
  return b;
}
int rounds_for(int key_bits) { return ceil_div(key_bits, kHistBits); }

void round_params(int key_bits, int r, int& hi, int& shift, int& width) {
  hi = key_bits - kHistBits * r;
  shift = hi - kHistBits > 0 ? hi - kHistBits : 0;
  width = hi - shift;
}

int launch_select_init(SelectState st, int nq, int64_t teff, cudaStream_t s) {
  select_init_kernel<<<ceil_div(nq, 256), 256, 0, s>>>(st, nq, teff);
  BVSS_TRY(post_launch(__func__, s));
  return BVSS_OK;
}

int launch_select_hist(int key_size, const void* keys, int64_t key_stride, int64_t n, int nq, SelectState st,
                       int key_bits, int r, int32_t* hist, cudaStream_t s) {
  int hi, shift, width;
  round_params(key_bits, r, hi, shift, width);
  const int hi_eff = (r == 0) ? 32 : hi;  // round 0: every key is in range
  const size_t smem = static_cast<size_t>(8) * (1u << width) * 4;
  if (key_size == 2) {
    auto kfn = select_hist_kernel<uint16_t>;
    BVSS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kfn<<<nq, 256, smem, s>>>(static_cast<const uint16_t*>(keys), key_stride, n, st, hi_eff, shift, width, hist);
  } else {
    auto kfn = select_hist_kernel<uint32_t>;
    BVSS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kfn<<<nq, 256, smem, s>>>(static_cast<const uint32_t*>(keys), key_stride, n, st, hi_eff, shift, width, hist);
  }
  BVSS_TRY(post_launch(__func__, s));
  return BVSS_OK;
}

int launch_select_resolve(const int32_t* hist, SelectState st, int nq, int key_bits, int r, cudaStream_t s) {
  int hi, shift, width;
  round_params(key_bits, r, hi, shift, width);
  const int last = (shift == 0) ? 1 : 0;
  select_resolve_kernel<<<ceil_div(nq, 8), 256, 0, s>>>(hist, st, nq, width, last);
  BVSS_TRY(post_launch(__func__, s));
  return BVSS_OK;
}

int launch_select_quota(SelectState st, const int64_t* all_eq, int nq, int world, int rank, cudaStream_t s) {
  select_quota_kernel<<<ceil_div(nq, 256), 256, 0, s>>>(st, all_eq, nq, world, rank);
  BVSS_TRY(post_launch(__func__, s));
  return BVSS_OK;
}

int launch_select_tiecount(const int32_t* local_hist, SelectState st, int nq, int64_t* eq_out, cudaStream_t s) {
  select_tiecount_kernel<<<ceil_div(nq, 256), 256, 0, s>>>(local_hist, st, nq, eq_out);
  BVSS_TRY(post_launch(__func__, s));
  return BVSS_OK;
}

int launch_select_bitmap(int key_size, const void* keys, int64_t key_stride, int64_t n, int nq, SelectState st,
                         int T, uint32_t* bitmap, int64_t words, cudaStream_t s, uint32_t key_limit) {
  if (key_size == 2)
    select_bitmap_kernel<uint16_t><<<nq, 256, 0, s>>>(static_cast<const uint16_t*>(keys), key_stride, n, st, T, bitmap,
                                                      words, key_limit);
  else
    select_bitmap_kernel<uint32_t><<<nq, 256, 0, s>>>(static_cast<const uint32_t*>(keys), key_stride, n, st, T, bitmap,
                                                      words, key_limit);
  BVSS_TRY(post_launch(__func__, s));
  return BVSS_OK;
}

int launch_select_emit(int key_size, const void* keys, int64_t key_stride, int64_t n, int nq, SelectState st, int T,
                       int64_t id_base, int32_t* cand, int32_t* score, int32_t* count, cudaStream_t s,
                       uint32_t key_limit) {
  if (key_size == 2)
    select_emit_kernel<uint16_t><<<nq, 256, 0, s>>>(static_cast<const uint16_t*>(keys), key_stride, n, st, T, id_base,
                                                    cand, score, count, key_limit);
  else
    select_emit_kernel<uint32_t><<<nq, 256, 0, s>>>(static_cast<const uint32_t*>(keys), key_stride, n, st, T, id_base,
                                                    cand, score, count, key_limit);
  BVSS_TRY(post_launch(__func__, s));
  return BVSS_OK;
}

// ------------------------------------------------ sampled-threshold path --
// The fused scan (scan_tc.cu, EMIT) appends every (id, key) with key <= tau_hat[q]
// to a per-query buffer, tau_hat being an order statistic of a strided sample of
// the database chosen so that, with overwhelming probability, at least T database
// keys are <= tau_hat.  This kernel then selects, exactly, the teff smallest
// (key, id) pairs of the buffer: an MSB radix select over the key (the teff-th
// key tau), a second radix select over the ids tied at tau (the quota-th id), and
// a compaction.  The result equals the full select's set because every key <= the
// true T-th key is in the buffer whenever cnt >= teff; a buffer with cnt < teff
// (the sample threshold was too low) or cnt > cap (overflow) is reported in
// `fail` and the caller redoes the batch on the full key path.  One CTA per query.
constexpr int kBufThreads = 512;

__device__ __forceinline__ void buf_radix_round(const uint32_t* __restrict__ vals, const uint32_t* __restrict__ keys,
                                                bool tie_filter, uint32_t tau, int c, int hi, int shift,
                                                uint32_t prefix, uint32_t* hist, int nbins) {
  const uint32_t mask = static_cast<uint32_t>(nbins) - 1u;
  for (int e = threadIdx.x; e < c; e += blockDim.x) {
    const uint32_t v = vals[e];
    const bool in = (!tie_filter || keys[e] == tau) && ((hi >= 32) || (v >> hi) == prefix);
    if (in) atomicAdd(&hist[(v >> shift) & mask], 1u);
  }
}

// one warp: first digit where the running count reaches need; returns (digit, count before it)
__device__ __forceinline__ void buf_find_digit(const uint32_t* hist, int nbins, uint32_t need, uint32_t* out_digit,
                                               uint32_t* out_before) {
  const int lane = threadIdx.x & 31;
  uint32_t run = 0;
  for (int b0 = 0; b0 < nbins; b0 += 32) {
    const int b = b0 + lane;
    const uint32_t v = b < nbins ? hist[b] : 0u;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, b < nbins && run + inc >= need);
    if (hit) {
      const int src = __ffs(hit) - 1;
      const uint32_t before = run + __shfl_sync(0xffffffffu, inc - v, src);
      if (lane == 0) {
        *out_digit = static_cast<uint32_t>(b0 + src);
        *out_before = before;
      }
      return;
    }
    run += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) {  // unreachable when need <= count in range
    *out_digit = static_cast<uint32_t>(nbins - 1);
    *out_before = run;
  }
}

// radix select of the need-th smallest value (1-based) among the (filtered) entries
__device__ uint32_t buf_select(const uint32_t* vals, const uint32_t* keys, bool tie_filter, uint32_t tau, int c,
                               int bits, uint32_t need, uint32_t* hist, uint32_t* s_dig, uint32_t* s_before,
                               uint32_t* need_left) {
  uint32_t prefix = 0;
  for (int hi = bits; hi > 0;) {
    const int shift = hi - kHistBits > 0 ? hi - kHistBits : 0;
    const int width = hi - shift;
    const int nbins = 1 << width;
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) hist[b] = 0u;
    __syncthreads();
    buf_radix_round(vals, keys, tie_filter, tau, c, hi, shift, prefix, hist, nbins);
    __syncthreads();
    if (threadIdx.x < 32) buf_find_digit(hist, nbins, need, s_dig, s_before);
    __syncthreads();
    prefix = (prefix << width) | *s_dig;
    need -= *s_before;
    __syncthreads();
    hi = shift;
  }
  *need_left = need;
  return prefix;
}

// power-of-two length of the in-smem id sort of select_buf_kernel (0: too long, not sorted)
__host__ __device__ __forceinline__ int sorted_len(int teff) {
  int p = 1;
  while (p < teff) p <<= 1;
  return p <= 16384 ? p : 0;
}

__global__ void __launch_bounds__(kBufThreads) select_buf_kernel(const int32_t* __restrict__ cnt,
                                                                 const uint32_t* __restrict__ bkey,
                                                                 const int32_t* __restrict__ bid, int cap, int teff,
                                                                 int key_bits, int T, int32_t* __restrict__ cand,
                                                                 int32_t* __restrict__ count, int* __restrict__ fail) {
  __shared__ uint32_t hist[kHistBins];
  __shared__ uint32_t s_dig, s_before, s_pos;
  const int q = blockIdx.x;
  const int c = cnt[q];
  int32_t* crow = cand + static_cast<int64_t>(q) * T;
  if (c < teff || c > cap) {
    if (threadIdx.x == 0) {
      atomicAdd(fail, 1);
      count[q] = 0;
    }
    return;
  }
  const uint32_t* keys = bkey + static_cast<int64_t>(q) * cap;
  const uint32_t* ids = reinterpret_cast<const uint32_t*>(bid + static_cast<int64_t>(q) * cap);
  uint32_t quota;
  const uint32_t tau = buf_select(keys, keys, false, 0u, c, key_bits, static_cast<uint32_t>(teff), hist, &s_dig,
                                  &s_before, &quota);
  // quota >= 1 ties at tau are taken, lowest ids first (reading R4)
  uint32_t dummy;
  const uint32_t theta = buf_select(ids, keys, true, tau, c, 31, quota, hist, &s_dig, &s_before, &dummy);
  if (threadIdx.x == 0) s_pos = 0u;
  __syncthreads();
  // the selected ids, then a bitonic sort so the list comes out in ascending id order (as the full-key path
  // and bvss_filter); lists longer than the smem sort stay in emission order (the refine then runs query-major)
  extern __shared__ uint32_t sort_buf[];
  const int P = sorted_len(teff);
  uint32_t* dst = P ? sort_buf : reinterpret_cast<uint32_t*>(crow);
  for (int e = threadIdx.x; e < c; e += blockDim.x) {
    const uint32_t k = keys[e];
    if (k < tau || (k == tau && ids[e] <= theta)) {
      const uint32_t pos = atomicAdd(&s_pos, 1u);
      dst[pos] = ids[e];
    }
  }
  if (P) {
    for (int i = teff + threadIdx.x; i < P; i += blockDim.x) sort_buf[i] = 0xFFFFFFFFu;
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
          const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
          const bool up = (lo & size) == 0;
          const uint32_t x = sort_buf[lo], y = sort_buf[hi];
          if ((x > y) == up) {
            sort_buf[lo] = y;
            sort_buf[hi] = x;
          }
        }
        __syncthreads();
      }
    }
    for (int i = threadIdx.x; i < teff; i += blockDim.x) crow[i] = static_cast<int32_t>(sort_buf[i]);
  }
  for (int i = teff + threadIdx.x; i < T; i += blockDim.x) crow[i] = -1;
  if (threadIdx.x == 0) count[q] = teff;
}

// strided database sample for the threshold estimate: sample j <- set floor(j n / ns)
__global__ void gather_sample_kernel(const uint4* __restrict__ sk, const int32_t* __restrict__ mass, int64_t n,
                                     int cps, int64_t ns, uint4* __restrict__ out, int32_t* __restrict__ out_mass) {
  const int64_t total = ns * cps;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t ch = t / ns, j = t % ns;
    const int64_t i = j * n / ns;
    out[ch * ns + j] = sk[ch * n + i];
    if (ch == 0) out_mass[j] = mass[i];
  }
}

bool select_buf_sorted(int teff) { return sorted_len(teff) != 0; }

int launch_select_buf(const int32_t* cnt, const uint32_t* bkey, const int32_t* bid, int cap, int teff, int key_bits,
                      int T, int nq, int32_t* cand, int32_t* count, int* fail, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(sorted_len(teff)) * 4;
  BVSS_CUDA(cudaFuncSetAttribute(select_buf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  select_buf_kernel<<<nq, kBufThreads, smem, s>>>(cnt, bkey, bid, cap, teff, key_bits, T, cand, count, fail);
  BVSS_TRY(post_launch(__func__, s));
  return BVSS_OK;
}

int launch_gather_sample(const void* sk, const int32_t* mass, int64_t n, int cps, int64_t ns, void* out,
                         int32_t* out_mass, int num_sms, cudaStream_t s) {
  gather_sample_kernel<<<num_sms * 4, 256, 0, s>>>(static_cast<const uint4*>(sk), mass, n, cps, ns,
                                                   static_cast<uint4*>(out), out_mass);
  BVSS_TRY(post_launch(__func__, s));
  return BVSS_OK;
}

}  // namespace bvss
