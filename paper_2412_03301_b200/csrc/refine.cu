// refine.cu — K5: Hausdorff refinement of the T candidates of every query on the
// 5th-generation tensor cores (Alg 6 lines 19-22; Def 4).
//
// For a query Q (m_q vectors) and a run of its candidate sets, the candidate
// vectors are gathered row by row into 128-row tiles (sets packed back to back,
// a set may straddle tiles) and the Gram matrix G = V Q^T is formed by
// tcgen05.mma (M = 128 candidate rows, N = m_q rounded up to 16, K = d) with an
// fp32 accumulator in TMEM.  Operands are the bf16 split x = hi + lo prepared at
// build time; terms = 3 issues hi*hi + hi*lo + lo*hi (|error| ~ 3 * 2^-18 |x||y|),
// terms = 1 issues hi*hi only.  The fused epilogue reads the accumulator with
// tcgen05.ld and forms D^2 = |v|^2 + |q|^2 - 2g (clamped at 0), the row minima
// (min over q, per candidate vector), the segmented column minima (min over the
// vectors of one set, per q), and per set
//     H^2 = max( max_q min_v D^2 , max_v min_q D^2 )
// (min/max on squared distances; sqrt is monotone).  K6 then recomputes the
// final top-k window exactly in fp32 (topk.cu).
//
// CTA = 9 warps: warps 0-3 gather (cp.async, SW128 layout, multi-stage ring),
// warps 4-7 epilogue (TMEM lanes 0-127 = tile rows), warp 8 owns TMEM and
// issues the MMAs from one thread.  Accumulators are double-buffered in TMEM so
// the epilogue of tile i overlaps the MMAs of tile i+1.  Persistent CTAs pull
// work items (query, up to 128 candidates) from an atomic counter.
#include "tc.cuh"

namespace bvss {

constexpr int kRows = 128;
constexpr int kItemCands = 128;
constexpr int kKChunk = 64;  // bf16 per K-chunk = 128 bytes = one SW128 row
constexpr int kProd = 128, kEpi = 128;
constexpr int kRefineThreads = kProd + kEpi + 32;
constexpr int kMaxN = 256;

struct RefineArgs {
  const __nv_bfloat16* hi;
  const __nv_bfloat16* lo;
  const float* vnorm;
  const int64_t* off;
  int dpad;
  const __nv_bfloat16* qhi;
  const __nv_bfloat16* qlo;
  const float* qnorm;
  const int64_t* qoff;
  const int32_t* cand;   // [nq][T] global ids (-1 padded)
  const int32_t* count;  // [nq] valid candidates per query (may be null: T)
  int T;
  int nq;
  int64_t id_base;
  float* out_h2;  // [nq][T]
  int terms;
  int nmax;        // max padded N over the batch
  int stages;
  uint32_t stage_bytes;
  uint32_t a_bytes;  // bytes of one A piece (16 KB)
  uint32_t b_bytes;  // bytes of one B piece (nmax * 128)
  uint32_t tmem_cols_per_acc;
  int items_per_query;
  int total_items;
  int* work_counter;
  unsigned long long* rows_counter;  // candidate rows gathered (stats)
};

struct RefineSmem {  // small control block after the stage ring
  float dsm[kRows][33];
  float carry_r[2][kMaxN];  // double-buffered by tile parity: read [t&1], write [(t+1)&1]
  float qn[kMaxN];
  uint32_t hq2s[kRows];
  float csm[kRows];
  int32_t rowstart[kItemCands + 1];
  int64_t vbase[kItemCands];
  uint64_t full[4];
  uint64_t empty[4];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  int item;
  float carry_h[2];
};

__device__ __forceinline__ int upper_bound_rows(const int32_t* rs, int nc, int R) {
  // largest c in [0, nc) with rs[c] <= R  (rs[0] = 0, strictly increasing)
  int lo = 0, hi = nc;  // invariant: rs[lo] <= R < rs[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (rs[mid] <= R) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kRefineThreads, 1) refine_tc_kernel(RefineArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align the stage ring (SW128 atoms)
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  RefineSmem& S = *reinterpret_cast<RefineSmem*>(ring + static_cast<size_t>(a.stages) * a.stage_bytes);
  const uint32_t ring_s = smem_u32(ring);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NST = a.stages;

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&S.full[s], kProd);
      tc::mbar_init(&S.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&S.tfull[b], 1);
      tc::mbar_init(&S.tempty[b], kEpi);
    }
    tc::fence_mbar_init();
  }
  if (warp == 8) tc::tmem_alloc(&S.tmem_base, 2 * a.tmem_cols_per_acc);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = S.tmem_base;

  // pipeline counters (identical sequence in every role)
  uint32_t kchunk_ctr = 0;  // global K-chunk counter (stage ring)
  uint32_t tile_ctr = 0;    // global tile counter (TMEM double buffer)
  const int KC = a.dpad / kKChunk;
  const uint32_t pieceA = a.a_bytes, pieceB = a.b_bytes;
  const bool three = a.terms == 3;

  for (;;) {
    if (tid == 0) S.item = atomicAdd(a.work_counter, 1);
    __syncthreads();
    const int item = S.item;
    if (item >= a.total_items) break;
    const int q = item / a.items_per_query;
    const int c0 = (item % a.items_per_query) * kItemCands;
    const int cnt = a.count ? a.count[q] : a.T;
    const int nc = min(kItemCands, cnt - c0);
    if (nc <= 0) {
      __syncthreads();
      continue;
    }
    const int64_t q0 = a.qoff[q];
    const int mq = static_cast<int>(a.qoff[q + 1] - q0);
    const int Nq = (mq + 15) & ~15;
    // ---- item table: sizes -> exclusive prefix (warps 0-3), query norms
    if (tid < kItemCands) {
      int sz = 0;
      if (tid < nc) {
        const int64_t cid = static_cast<int64_t>(a.cand[static_cast<int64_t>(q) * a.T + c0 + tid]) - a.id_base;
        const int64_t b = a.off[cid];
        sz = static_cast<int>(a.off[cid + 1] - b);
        S.vbase[tid] = b;
      }
      // block-wide inclusive scan over 128 threads (4 warps) via shuffles + smem
      int inc = sz;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      if (lane == 31) S.rowstart[warp] = inc;  // temp: warp totals
      tc::named_bar(1, kItemCands);
      int wpre = 0;
      for (int w = 0; w < warp; ++w) wpre += S.rowstart[w];
      tc::named_bar(1, kItemCands);
      S.rowstart[tid + 1] = wpre + inc;
      if (tid == 0) S.rowstart[0] = 0;
    }
    for (int j = tid; j < kMaxN; j += blockDim.x) S.qn[j] = (j < mq) ? a.qnorm[q0 + j] : 0.0f;
    for (int j = tid; j < kRows; j += blockDim.x) S.hq2s[j] = 0u;
    __syncthreads();
    const int total_rows = S.rowstart[nc];
    const int ntiles = (total_rows + kRows - 1) / kRows;
    if (tid == 0 && a.rows_counter) atomicAdd(a.rows_counter, static_cast<unsigned long long>(total_rows));

    if (warp < 4) {
      // =========================== producers: cp.async gather ===========================
      const int u = tid & 7, rsub = tid >> 3;  // 16-byte chunk within the 128-byte row; row group
      const int lag = NST - 1;
      uint32_t first_pending = kchunk_ctr;  // oldest K-chunk not yet signalled
      for (int tile = 0; tile < ntiles; ++tile) {
        int64_t vrow[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int R = tile * kRows + rsub + 16 * i;
          if (R < total_rows) {
            const int c = upper_bound_rows(S.rowstart, nc, R);
            vrow[i] = S.vbase[c] + (R - S.rowstart[c]);
          } else {
            vrow[i] = -1;
          }
        }
        for (int kc = 0; kc < KC; ++kc) {
          const uint32_t st = kchunk_ctr % NST;
          tc::mbar_wait(&S.empty[st], ((kchunk_ctr / NST) & 1u) ^ 1u);
          const uint32_t sbase = ring_s + st * a.stage_bytes;
          const uint32_t a_hi = sbase, a_lo = sbase + pieceA;
          const uint32_t b_hi = sbase + (three ? 2 : 1) * pieceA, b_lo = b_hi + pieceB;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = rsub + 16 * i;
            const uint32_t o = tc::sw128_off(r, u);
            const int64_t v = vrow[i];
            const size_t e = (v >= 0 ? static_cast<size_t>(v) : 0) * a.dpad + kc * kKChunk + u * 8;
            const uint32_t nb = v >= 0 ? 16u : 0u;
            tc::cp_async16(a_hi + o, a.hi + e, nb);
            if (three) tc::cp_async16(a_lo + o, a.lo + e, nb);
          }
          for (int j = rsub; j < Nq; j += 16) {
            const uint32_t o = tc::sw128_off(j, u);
            const bool ok = j < mq;
            const size_t e = static_cast<size_t>(ok ? q0 + j : 0) * a.dpad + kc * kKChunk + u * 8;
            tc::cp_async16(b_hi + o, a.qhi + e, ok ? 16u : 0u);
            if (three) tc::cp_async16(b_lo + o, a.qlo + e, ok ? 16u : 0u);
          }
          tc::cp_async_commit();
          ++kchunk_ctr;
          // signal chunks that are at least `lag` groups old
          while (kchunk_ctr - first_pending > static_cast<uint32_t>(lag)) {
            if (lag >= 3) tc::cp_async_wait<3>();
            else if (lag == 2) tc::cp_async_wait<2>();
            else tc::cp_async_wait<1>();
            tc::fence_proxy_async_smem();
            tc::mbar_arrive(&S.full[first_pending % NST]);
            ++first_pending;
          }
        }
      }
      tc::cp_async_wait<0>();
      tc::fence_proxy_async_smem();
      while (first_pending != kchunk_ctr) {
        tc::mbar_arrive(&S.full[first_pending % NST]);
        ++first_pending;
      }
    } else if (warp == 8) {
      // =========================== MMA issuer (one thread) ===========================
      const uint32_t idesc = tc::idesc_bf16_f32(kRows, Nq);
      for (int tile = 0; tile < ntiles; ++tile) {
        const uint32_t acc = tile_ctr & 1u;
        tc::mbar_wait(&S.tempty[acc], ((tile_ctr >> 1) & 1u) ^ 1u);
        tc::fence_after_sync();
        const uint32_t d_tmem = tmem + acc * a.tmem_cols_per_acc;
        for (int kc = 0; kc < KC; ++kc) {
          const uint32_t st = kchunk_ctr % NST;
          tc::mbar_wait(&S.full[st], (kchunk_ctr / NST) & 1u);
          tc::fence_after_sync();
          if (lane == 0) {
            const uint32_t sbase = ring_s + st * a.stage_bytes;
            const uint32_t a_hi = sbase, a_lo = sbase + pieceA;
            const uint32_t b_hi = sbase + (three ? 2 : 1) * pieceA, b_lo = b_hi + pieceB;
#pragma unroll
            for (int kk = 0; kk < kKChunk / 16; ++kk) {
              const uint32_t koff = kk * 32;
              const uint32_t accum = (kc | kk) ? 1u : 0u;
              tc::umma_bf16(d_tmem, tc::sw128_desc(a_hi + koff), tc::sw128_desc(b_hi + koff), idesc, accum);
              if (three) {
                tc::umma_bf16(d_tmem, tc::sw128_desc(a_hi + koff), tc::sw128_desc(b_lo + koff), idesc, 1u);
                tc::umma_bf16(d_tmem, tc::sw128_desc(a_lo + koff), tc::sw128_desc(b_hi + koff), idesc, 1u);
              }
            }
            tc::umma_commit(&S.empty[st]);
            if (kc == KC - 1) tc::umma_commit(&S.tfull[acc]);
          }
          __syncwarp();
          ++kchunk_ctr;
        }
        ++tile_ctr;
      }
    } else {
      // =========================== epilogue (warps 4-7) ===========================
      const int ew = warp - 4;
      const int r = ew * 32 + lane;  // tile row == TMEM lane
      const int et = tid - kProd;    // 0..127
      float* out = a.out_h2 + static_cast<int64_t>(q) * a.T + c0;
      for (int tile = 0; tile < ntiles; ++tile) {
        const uint32_t acc = tile_ctr & 1u;
        const int ts = tile * kRows;
        const int R = ts + r;
        const bool valid = R < total_rows;
        float vn = 0.0f;
        if (valid) {
          const int c = upper_bound_rows(S.rowstart, nc, R);
          vn = a.vnorm[S.vbase[c] + (R - S.rowstart[c])];
        }
        const int tile_end = min(total_rows, ts + kRows);
        const int cf = upper_bound_rows(S.rowstart, nc, ts);
        const int cl = upper_bound_rows(S.rowstart, nc, tile_end - 1);
        const int nseg = cl - cf + 1;
        const bool carry_in = S.rowstart[cf] < ts;
        const bool carry_out = S.rowstart[cl + 1] > tile_end;

        tc::mbar_wait(&S.tfull[acc], (tile_ctr >> 1) & 1u);
        tc::fence_after_sync();
        float cmin = __int_as_float(0x7f800000);
        const uint32_t tbase = tmem + acc * a.tmem_cols_per_acc + (static_cast<uint32_t>(ew * 32) << 16);
        for (int cc = 0; cc < Nq; cc += 32) {
          uint32_t g0[16], g1[16];
          tc::tmem_ld16(tbase + cc, g0);
          if (cc + 16 < Nq) tc::tmem_ld16(tbase + cc + 16, g1);
          tc::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = cc + j;
            const uint32_t gb = j < 16 ? g0[j] : g1[j - 16];
            float d2 = __int_as_float(0x7f800000);
            if (col < mq && valid) {
              const float g = __uint_as_float(gb);
              d2 = fmaxf(vn + S.qn[col] - 2.0f * g, 0.0f);
              cmin = fminf(cmin, d2);
            }
            S.dsm[r][j] = d2;
          }
          tc::named_bar(2, kEpi);
          // segmented column minima for columns cc .. cc+31
          for (int p = et; p < nseg * 32; p += kEpi) {
            const int s = p >> 5, j = p & 31, col = cc + j;
            if (col >= mq) continue;
            const int c = cf + s;
            const int rb = max(S.rowstart[c], ts) - ts, re = min(S.rowstart[c + 1], tile_end) - ts;
            float m = __int_as_float(0x7f800000);
            for (int rr = rb; rr < re; ++rr) m = fminf(m, S.dsm[rr][j]);
            if (s == 0 && carry_in) m = fminf(m, S.carry_r[tile & 1][col]);
            if (s == nseg - 1 && carry_out) S.carry_r[(tile + 1) & 1][col] = m;
            else atomicMax(&S.hq2s[s], __float_as_uint(m));
          }
          tc::named_bar(2, kEpi);
        }
        // accumulator fully read: hand the TMEM buffer back to the MMA warp
        tc::fence_before_sync();
        tc::mbar_arrive(&S.tempty[acc]);
        S.csm[r] = valid ? cmin : 0.0f;
        tc::named_bar(2, kEpi);
        if (et < nseg) {
          const int s = et, c = cf + s;
          const int rb = max(S.rowstart[c], ts) - ts, re = min(S.rowstart[c + 1], tile_end) - ts;
          float hv = 0.0f;
          for (int rr = rb; rr < re; ++rr) hv = fmaxf(hv, S.csm[rr]);
          if (s == 0 && carry_in) hv = fmaxf(hv, S.carry_h[tile & 1]);
          if (s == nseg - 1 && carry_out) {
            S.carry_h[(tile + 1) & 1] = hv;
          } else {
            const float hq = __uint_as_float(S.hq2s[s]);
            out[c] = fmaxf(hv, hq);
          }
          S.hq2s[s] = 0u;
        }
        tc::named_bar(2, kEpi);
        ++tile_ctr;
      }
    }
    // keep every role's counters in step (producers/MMA advanced kchunk_ctr, epilogue/MMA tile_ctr)
    if (warp < 4) tile_ctr += ntiles;
    else if (warp == 8) { /* both advanced */ }
    else kchunk_ctr += ntiles * KC;
    __syncthreads();
  }
  __syncthreads();
  if (warp == 8) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, 2 * a.tmem_cols_per_acc);
  }
}

size_t refine_smem_bytes(int terms, int nmax, int& stages, uint32_t& stage_bytes) {
  const uint32_t a_bytes = kRows * 128;
  const uint32_t b_bytes = static_cast<uint32_t>(nmax) * 128;
  stage_bytes = (terms == 3 ? 2u : 1u) * (a_bytes + b_bytes);
  stage_bytes = (stage_bytes + 1023u) & ~1023u;
  const size_t ctrl = (sizeof(RefineSmem) + 127) & ~size_t(127);
  const size_t budget = 227 * 1024 - 1024 - ctrl;
  stages = static_cast<int>(budget / stage_bytes);
  if (stages > 4) stages = 4;
  return static_cast<size_t>(stages) * stage_bytes + ctrl + 1024;
}

int launch_refine_tc(const __nv_bfloat16* hi, const __nv_bfloat16* lo, const float* vnorm, const int64_t* off,
                     int dpad, const __nv_bfloat16* qhi, const __nv_bfloat16* qlo, const float* qnorm,
                     const int64_t* qoff, int max_mq, const int32_t* cand, const int32_t* count, int T, int nq,
                     int64_t id_base, float* out_h2, int terms, int* work_counter,
                     unsigned long long* rows_counter, int num_sms, cudaStream_t st) {
  if (nq <= 0 || T <= 0) return BVSS_OK;
  if (max_mq > kMaxN) BVSS_FAIL(BVSS_EUNSUPPORTED, "query set with %d vectors exceeds the %d-row refine tile", max_mq, kMaxN);
  if (dpad % kKChunk) BVSS_FAIL(BVSS_EINVAL, "dpad must be a multiple of 64");
  RefineArgs a;
  a.hi = hi; a.lo = lo; a.vnorm = vnorm; a.off = off; a.dpad = dpad;
  a.qhi = qhi; a.qlo = qlo; a.qnorm = qnorm; a.qoff = qoff;
  a.cand = cand; a.count = count; a.T = T; a.nq = nq; a.id_base = id_base; a.out_h2 = out_h2;
  a.terms = terms == 1 ? 1 : 3;
  a.nmax = (max_mq + 15) & ~15;
  if (a.nmax < 16) a.nmax = 16;
  int stages;
  uint32_t stage_bytes;
  const size_t smem = refine_smem_bytes(a.terms, a.nmax, stages, stage_bytes);
  if (stages < 2) BVSS_FAIL(BVSS_EUNSUPPORTED, "refine tile does not fit shared memory");
  a.stages = stages;
  a.stage_bytes = stage_bytes;
  a.a_bytes = kRows * 128;
  a.b_bytes = static_cast<uint32_t>(a.nmax) * 128;
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(a.nmax)) cols <<= 1;
  a.tmem_cols_per_acc = cols;
  a.items_per_query = ceil_div(T, kItemCands);
  a.total_items = a.items_per_query * nq;
  a.work_counter = work_counter;
  a.rows_counter = rows_counter;
  BVSS_CUDA(cudaMemsetAsync(work_counter, 0, sizeof(int), st));
  BVSS_CUDA(cudaFuncSetAttribute(refine_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int grid = a.total_items < num_sms ? a.total_items : num_sms;
  refine_tc_kernel<<<grid, kRefineThreads, smem, st>>>(a);
  BVSS_TRY(post_launch(__func__, st));
  return BVSS_OK;
}

}  // namespace bvss
