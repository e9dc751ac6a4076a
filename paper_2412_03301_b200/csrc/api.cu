// api.cu — host runtime and C ABI of libbvss (include/bvss.h).
//
// Owns the index (device buffers, stream, workspace), validates arguments,
// generates the projection W (H2, reading R7), plans query sub-batches and
// launches the kernels of the hot path:
//   build : K1 encode (+K9 norms, fp16 split)  ->  K2 sketches
//   search: K1/K2 on the queries -> K3 scan -> K4 select -> K5 refine -> K6 top-k
#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace bvss {

// ---------------------------------------------------------------- errors --
static thread_local char g_err[1024] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int post_launch(const char* what, cudaStream_t st) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
    return BVSS_ECUDA;
  }
  static const bool dbg = [] {
    const char* v = getenv("BVSS_DEBUG_SYNC");
    return v && v[0] == '1';
  }();
  if (dbg) {
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      set_error("%s: kernel failed: %s", what, cudaGetErrorString(e));
      return BVSS_ECUDA;
    }
  }
  return BVSS_OK;
}

// kernels (other translation units)
int launch_encode(const float* V, int64_t nvec, int d, const uint16_t* Wt, int m, int s, int L, uint32_t* codes,
                  float* norms, __half* hs, __half* ls, float* scale, int dpad, int64_t rows, const int64_t* dst_row,
                  int kcs, int num_sms, cudaStream_t st);
int refine_kcs(int dpad);
int launch_finite_check(const float* x, int64_t count, int* bad_dev, int num_sms, cudaStream_t st);
int launch_sketch(const uint32_t* codes, int m, const int64_t* off, int64_t n, int kind, void* S, int32_t* mass,
                  int64_t cstride, int64_t sstride, int num_sms, cudaStream_t st);
int launch_unchunk(const void* S, int64_t n_stride, int64_t first, int64_t count, int words, uint32_t* out,
                   cudaStream_t st);
int launch_scan(int kind, const void* S, const int32_t* mass, int64_t n, int64_t n_stride, int m, const void* SQ,
                const int32_t* massQ, int nq, void* keys, int64_t key_stride, int num_sms, cudaStream_t st);
int launch_scan_tc(int kind, const void* S, const int32_t* mass, int64_t n, int64_t n_stride, int m, const void* SQ,
                   const int32_t* massQ, int nq, void* Qx, int qpad, void* keys, int64_t key_stride, int* work_counter,
                   int num_sms, cudaStream_t st, const uint32_t* tau, int32_t* cnt, int32_t* buf_id, uint32_t* buf_key,
                   int cap, int64_t id_base, bool expand);
int launch_select_buf(const int32_t* cnt, const uint32_t* bkey, const int32_t* bid, int cap, int teff, int key_bits,
                      int T, int nq, int32_t* cand, int32_t* count, int* fail, cudaStream_t s);
int launch_expand_db_fp4(const void* S, int64_t n, int64_t n_stride, int m, void* X, int num_sms, cudaStream_t st);
int scan_tc_units(int kind, int m);
uint64_t scan_tc_db_bytes(int kind, int m, int64_t n, int nq, int num_sms);
bool select_buf_sorted(int teff);
int launch_gather_sample(const void* sk, const int32_t* mass, int64_t n, int cps, int64_t ns, void* out,
                         int32_t* out_mass, int num_sms, cudaStream_t s);
struct SelectState {
  uint32_t* prefix;
  int64_t* below;
  int64_t* teff;
  int64_t* eq;
  int64_t* quota;
  int32_t* digit;
};
int key_bits_for(int kind, int m);
int rounds_for(int key_bits);
int launch_select_init(SelectState st, int nq, int64_t teff, cudaStream_t s);
int launch_select_hist(int key_size, const void* keys, int64_t key_stride, int64_t n, int nq, SelectState st,
                       int key_bits, int r, int32_t* hist, cudaStream_t s);
int launch_select_resolve(const int32_t* hist, SelectState st, int nq, int key_bits, int r, cudaStream_t s);
int launch_select_quota(SelectState st, const int64_t* all_eq, int nq, int world, int rank, cudaStream_t s);
int launch_select_tiecount(const int32_t* local_hist, SelectState st, int nq, int64_t* eq_out, cudaStream_t s);
int launch_select_emit(int key_size, const void* keys, int64_t key_stride, int64_t n, int nq, SelectState st, int T,
                       int64_t id_base, int32_t* cand, int32_t* score, int32_t* count, cudaStream_t s,
                       uint32_t key_limit);
int launch_gate_planes(const void* S, int64_t n, int m, int kind, int M, uint32_t* planes, int64_t W, int num_sms,
                       cudaStream_t st);
int launch_gate_positions(const uint32_t* qcodes, const int64_t* qoff, int nq, int m, int A, int32_t* pos,
                          cudaStream_t st);
int launch_gate_keys(int key_size, void* keys, int64_t key_stride, int64_t n, int nq, const int32_t* pos, int A,
                     const uint32_t* planes, int64_t W, int num_sms, cudaStream_t st);
int launch_alg2_keys(const uint32_t* qcodes, const int64_t* qoff, int nq, int max_mq, const uint32_t* codes,
                     const int64_t* off, int64_t n, int m, uint16_t* keys, int64_t key_stride, int num_sms,
                     cudaStream_t st);
int launch_refine_tc(const __half* hs, const __half* ls, const float* vscale, int64_t prows, const int64_t* pbase,
                     const float* vnorm, const int64_t* off, int dpad, const __half* qhs, const __half* qls,
                     const float* qscale, int64_t qrows, const int64_t* qrow, const float* qnorm, const int64_t* qoff, int max_mq, const int32_t* cand,
                     const int32_t* count, int T, int nq, int64_t id_base, float* out_h2, int terms, int* work_counter,
                     unsigned long long* rows_counter, int num_sms, int64_t n_local, int32_t* bounds, int metric,
                     float* out_err, float c1, float c2, float vmax2, cudaStream_t st);
int64_t refine_range_sets(int64_t n_local, int64_t prows, int dpad, int T);
int launch_topk_fixup(const float* approx, const int32_t* cand, const int32_t* count, int T, int k, const float* V,
                      const int64_t* off, int64_t id_base, int d, const float* Qv, const int64_t* qoff,
                      const float* qnorm, float vmax2, float c1, float c2, int exact_all, int64_t* out_ids,
                      float* out_dist, int nq, int64_t* fixup_counter, void* scratch, int metric,
                      const float* approx_err, int max_rows, int max_mq, cudaStream_t st);
int launch_merge_topk(const int64_t* ids, const float* dist, int P, int64_t nq, int k, int64_t* out_ids,
                      float* out_dist, cudaStream_t st);
int launch_select_bitmap(int key_size, const void* keys, int64_t key_stride, int64_t n, int nq, SelectState st,
                         int T, uint32_t* bitmap, int64_t words, cudaStream_t s, uint32_t key_limit);
int dense_max_dpad();
int dense_epi_sub();
int dense_tile_rows();
int launch_dense_db_operand(const float* V, int64_t nvec, int d, int dpad, float inv_s, __half* hd, int num_sms,
                            cudaStream_t st);
int launch_dense_query_operand(const float* Qv, const float* qnorm, const int32_t* rowmap, const int32_t* rowq,
                               int64_t rows, int d, int dpad, float inv_s, __half* qd, int32_t* lane_qid,
                               float* lane_qn, int num_sms, cudaStream_t st);
int launch_dense_prep(const int64_t* qoff, const float* qnorm, int nq, float c1, float c2, float vmax2, float* qE,
                      float* lists, int64_t nlist, int32_t* cnt, const int32_t* huge, int nhuge, const uint32_t* mask,
                      int64_t mask_stride, int64_t id_base, int32_t* ids, float* vals, int cap, int num_sms,
                      cudaStream_t st);
int launch_dense_norm_operand(const float* vn, int64_t nvec, float inv_s2, __half* va, int num_sms, cudaStream_t st);
int launch_dense_hausdorff(const __half* qd, int ntq, const __half* hd, int64_t nvec, int dpad, int ntiles,
                           const int32_t* tile_s0, const int32_t* tile_s1, const int64_t* off, const __half* va,
                           const __half* qa, const int32_t* lane_qid, const float* lane_qn, const float* qE,
                           float* tau0,
                           float kappa, float alpha, int k, int R, float* lists, int32_t* cnt, int32_t* ids,
                           float* vals, int cap,
                           const uint32_t* mask, int64_t mask_stride, int64_t id_base, unsigned long long* stat,
                           int dyn, int* unit_ctr, int* udone, int num_sms, cudaStream_t st);

// ------------------------------------------------------- small kernels --
__global__ void fill_i32_kernel(int32_t* __restrict__ x, int64_t n, int32_t v) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) x[i] = v;
}
__global__ void fill_f32_kernel(float* __restrict__ x, int64_t n, float v) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) x[i] = v;
}
void fill_f32_inf(float* x, int64_t n, cudaStream_t st) {
  if (n > 0) fill_f32_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, st>>>(x, n, INFINITY);
}
__global__ void max_float_kernel(const float* __restrict__ x, int64_t n, unsigned int* __restrict__ out) {
  float m = 0.0f;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m = fmaxf(m, x[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));  // values >= 0
}
// padded refine row of every DB vector: set i's rows start at pbase[i] (8-aligned)
__global__ void pad_rows_kernel(const int64_t* __restrict__ off, const int64_t* __restrict__ pbase, int64_t n,
                                int64_t* __restrict__ dst_row) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    for (int64_t v = off[i]; v < off[i + 1]; ++v) dst_row[v] = pbase[i] + (v - off[i]);
}
__global__ void count_valid_kernel(const int32_t* __restrict__ cand, int T, int nq, int32_t* __restrict__ count) {
  const int q = blockIdx.x;
  int c = 0;
  for (int i = threadIdx.x; i < T; i += blockDim.x) c += cand[static_cast<int64_t>(q) * T + i] >= 0 ? 1 : 0;
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ int s[8];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) t += s[w];
    count[q] = t;
  }
}

// candidate rows of one brute-force chunk: cand[q][i] = c0 + i (i < cnt), count[q] = cnt
__global__ void fill_range_kernel(int32_t* __restrict__ cand, int32_t* __restrict__ count, int nq, int T, int64_t c0,
                                  int cnt) {
  const int64_t total = static_cast<int64_t>(nq) * T;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(t % T);
    cand[t] = i < cnt ? static_cast<int32_t>(c0 + i) : -1;
    if (i == 0) count[t / T] = cnt;
  }
}

// ------------------------------------------------------------ workspace --
struct Workspace {
  std::map<std::string, std::pair<void*, size_t>> bufs;
  size_t total = 0;
  int get(const char* name, size_t bytes, void** out) {
    auto it = bufs.find(name);
    if (it != bufs.end() && it->second.second >= bytes) {
      *out = it->second.first;
      return BVSS_OK;
    }
    if (it != bufs.end()) {
      cudaFree(it->second.first);
      total -= it->second.second;
      bufs.erase(it);
    }
    void* p = nullptr;
    const size_t b = bytes < 256 ? 256 : bytes;
    BVSS_CUDA(cudaMalloc(&p, b));
    bufs[name] = {p, b};
    total += b;
    *out = p;
    return BVSS_OK;
  }
  void release() {
    for (auto& kv : bufs) cudaFree(kv.second.first);
    bufs.clear();
    total = 0;
  }
};

// ------------------------------------------------------------ projection --
// H2: W from the seed, reading R7 (SplitMix64 per row, rejection of the
// modulo-biased tail, distinct dims, sorted).  Independent of the oracle.
static uint64_t splitmix_next(uint64_t& x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static void make_projection(uint64_t seed, int m, int s, int d, std::vector<uint16_t>& W) {
  W.assign(static_cast<size_t>(m) * s, 0);
  const uint64_t r = (0ull - static_cast<uint64_t>(d)) % static_cast<uint64_t>(d);  // 2^64 mod d
  for (int j = 0; j < m; ++j) {
    uint64_t x = seed ^ (static_cast<uint64_t>(j) * 0xD1B54A32D192ED03ull);
    std::vector<int> chosen;
    while (static_cast<int>(chosen.size()) < s) {
      const uint64_t u = splitmix_next(x);
      if (r != 0 && u >= 0ull - r) continue;  // u >= 2^64 - r
      const int i = static_cast<int>(u % static_cast<uint64_t>(d));
      bool dup = false;
      for (int c : chosen) dup |= (c == i);
      if (!dup) chosen.push_back(i);
    }
    std::sort(chosen.begin(), chosen.end());
    for (int t = 0; t < s; ++t) W[static_cast<size_t>(j) * s + t] = static_cast<uint16_t>(chosen[t]);
  }
}

}  // namespace bvss

using namespace bvss;

struct bvss_index {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  int num_sms = 148;
  int64_t n = 0, nvec = 0;
  int d = 0, dpad = 0;
  int max_rows = 0;             // largest set (rows): selects the packed K6 variant
  uint32_t m = 0, s = 0, L = 0, sketch = 0;
  uint64_t seed = 0;
  int terms = 3;
  uint32_t query_batch = 0;
  std::vector<uint16_t> W;    // [m][s]
  uint16_t* Wt = nullptr;     // device [s][m]
  float* V = nullptr;         // [nvec][d]
  int64_t* off = nullptr;     // [n+1]
  __half* hi = nullptr;         // [dpad/64][prows][64] chunk-major, pre-swizzled, 8-aligned sets (refine.cu)
  __half* lo = nullptr;
  float* vscale = nullptr;      // [prows] power-of-two scale of each row
  int64_t prows = 0;            // padded refine rows
  int64_t* pbase = nullptr;     // [n+1] first padded row of each set
  float* vnorm = nullptr;
  float vmax2 = 0.0f;
  uint32_t* codes = nullptr;  // optional [nvec][m/32]
  void* sk = nullptr;         // chunk-major sketches
  int32_t* mass = nullptr;
  uint32_t select_mode = 0;   // 0 auto, 1 full keys, 2 sampled threshold
  int metric = 0;             // rerank metric: 0 Hausdorff, 1 MeanMin, 2 Min (bvss_params.metric)
  int score = 0;              // filter score: 0 Hamming / L2^2, 1 OVERLAP (bvss_params.score, reading R24)
  int64_t ns = 0;             // database sample for the threshold estimate (select_mode 2)
  void* smp_sk = nullptr;     // chunk-major sketches of the sample
  void* skx = nullptr;        // binary: tensor-core scan operand, FP4 expansion [m/32][n][16 B] (scan_tc.cu)
  void* smp_skx = nullptr;    // the same for the sample
  int32_t* smp_mass = nullptr;
  size_t owned_bytes = 0;
  // streaming build (bvss_index_begin / append / finish): vectors land in pend_V until finish
  bool pending = false;
  int64_t n_total = 0, nvec_total = 0, n_appended = 0, nvec_appended = 0;
  std::vector<int64_t> pend_off;
  std::vector<uint16_t> pend_proj;
  bvss_params pend_p{};
  float* pend_V = nullptr;
  // candidate generation variants (gate.cu): BioVSS++ stage 1 (A, M) and BioVSS Alg 2
  uint32_t gate_A = 0, gate_M = 0;  // stage-1 gate: A query positions, minimum count M (A = 0: open)
  uint32_t filter = 0;              // 0 = sketch scan (Alg 6), 1 = Haus^H over per-vector codes (Alg 2)
  uint32_t* planes = nullptr;       // [m][ceil(n/32)] gate bit planes
  int64_t gW = 0;
  // dense (candidate-major) refine, dense.cu: built on first use
  std::vector<int64_t> off_h;   // host copy of the set offsets
  __half* hd = nullptr;         // [nvec][dpad] fp16 = x / dense_s
  __half* va = nullptr;         // [nvec][16] fp16: the split |v|^2 / dense_s^2 (the MMA's norm chunk)
  float dense_s = 1.0f;         // power of two >= max|x|
  int32_t* dtile_s0 = nullptr;  // [dntiles] first set of each dense tile (whole sets, <= 256 rows)
  int32_t* dtile_s1 = nullptr;
  int dntiles = 0;
  std::vector<int32_t> dtile_s0_h;
  int32_t* dhuge = nullptr;     // sets of more than 256 rows (exact path)
  int dnhuge = 0;
  unsigned long long dense_stat[2] = {0, 0};  // survivors / emitted of the last dense call
  Workspace ws;
  bvss_stats stats{};
  cudaEvent_t ev[8] = {};
};

struct bvss_search_ctx {
  bvss_index* idx = nullptr;
  int64_t nq = 0;
  int k = 0, T = 0;
  int64_t teff = 0;
  int64_t id_base = 0;
  int key_bits = 0, rounds = 0, next_round = 0;
  int max_mq = 0;
  int64_t nqvec = 0;
  std::vector<int64_t> qoff_host;
  // device
  float* qv = nullptr;
  int64_t* qoff = nullptr;
  float* qnorm = nullptr;
  __half* qhi = nullptr;         // [dpad/64][qrows][64] chunk-major, pre-swizzled, 8-aligned queries
  __half* qlo = nullptr;
  float* qscale = nullptr;       // [qrows]
  int64_t qrows = 0;
  int64_t* qrow = nullptr;       // [nq] first padded row of each query
  void* keys = nullptr;
  int64_t key_stride = 0;
  void* qx = nullptr;         // expanded queries of the tensor-core scan
  int qpad = 0;
  SelectState sel{};
  int32_t* local_hist = nullptr;
  int32_t* cand = nullptr;
  int32_t* count = nullptr;
  bool cand_sorted = true;    // candidate lists in ascending id order (the refine may then run range-major)
  float* approx = nullptr;
  float* approx_err = nullptr; // MeanMin: per-candidate bound on |approx - exact| (refine.cu)
  void* qsk = nullptr;        // query sketches, row-major padded to whole chunks
  int32_t* qmass = nullptr;   // query sketch masses
  uint32_t* qcodes = nullptr; // query codes
  int32_t* gate_pos = nullptr; // [nq][gate_A] stage-1 positions of every query (gate.cu)
  int nalloc = 0;
  // buffers come from the index workspace (grow-only, reused across calls in the same order)
  int alloc(size_t bytes, void** p);
};

int bvss_search_ctx::alloc(size_t bytes, void** p) {
  const std::string name = "ctx" + std::to_string(nalloc++);
  return idx->ws.get(name.c_str(), bytes, p);
}

namespace {

int check_device(int dev, int* num_sms) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) BVSS_FAIL(BVSS_EUNSUPPORTED, "no CUDA device available (no CPU fallback)");
  if (dev < 0 || dev >= count) BVSS_FAIL(BVSS_EINVAL, "device %d out of range (%d visible)", dev, count);
  cudaDeviceProp p;
  BVSS_CUDA(cudaGetDeviceProperties(&p, dev));
  if (p.major != 10) BVSS_FAIL(BVSS_EUNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a", dev, p.major, p.minor);
  *num_sms = p.multiProcessorCount;
  return BVSS_OK;
}

int check_offsets(const int64_t* o, int64_t n, const char* what) {
  if (o[0] != 0) BVSS_FAIL(BVSS_EINVAL, "%s offsets must start at 0", what);
  for (int64_t i = 0; i < n; ++i)
    if (o[i + 1] <= o[i]) BVSS_FAIL(BVSS_EINVAL, "%s set %lld is empty or offsets decrease (Def 2: m >= 1)", what,
                                    static_cast<long long>(i));
  return BVSS_OK;
}

int to_device(bvss_index* idx, void* dst, const void* src, size_t bytes, bool dev_ptrs) {
  if (bytes == 0) return BVSS_OK;
  BVSS_CUDA(cudaMemcpyAsync(dst, src, bytes, dev_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, idx->stream));
  return BVSS_OK;
}
int from_device(bvss_index* idx, void* dst, const void* src, size_t bytes, bool dev_ptrs) {
  if (bytes == 0) return BVSS_OK;
  BVSS_CUDA(cudaMemcpyAsync(dst, src, bytes, dev_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, idx->stream));
  return BVSS_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// OVERLAP (R24) key offset: K0 - 2 <S_Q, S_i> >= 0 for every pair (binary: <.,.> <= m; count: <= m 255^2)
int64_t overlap_k0(const bvss_index* idx) {
  return idx->sketch == BVSS_SKETCH_BINARY ? 2ll * idx->m : 2ll * idx->m * 255 * 255;
}

bool gated(const bvss_index* idx) { return idx->gate_A > 0 && idx->gate_M > 0; }
// key rows: u16 for binary sketches and for Alg 2's Haus^H; u32 for count-sketch scores
int key_size_of(const bvss_index* idx) { return (idx->sketch == BVSS_SKETCH_BINARY || idx->filter == 1) ? 2 : 4; }
// keys at or above the limit are the stage-1 gate's rejects (their top bit set): never candidates
uint32_t key_limit_of(const bvss_index* idx) {
  if (!gated(idx)) return 0xFFFFFFFFu;
  return key_size_of(idx) == 2 ? 0x8000u : 0x80000000u;
}

int chunks_per_set(const bvss_index* idx) {
  return idx->sketch == BVSS_SKETCH_BINARY ? static_cast<int>(((idx->m / 32) + 3) / 4) : static_cast<int>(idx->m / 16);
}

// error-bound constants of the refine arithmetic: scaled fp16
// split, y = x/s with s a power of two >= max|x|, |y - fp16(y)| <= 2^-11|y| + 2^-25.
void error_consts(const bvss_index* idx, float* c1, float* c2) {
  const double u23 = std::ldexp(1.0, -23);
  const double dd = static_cast<double>(idx->dpad);
  const double sq = std::sqrt(dd);
  const int terms = idx->terms == 3 ? 3 : 1;
  const double prod = terms == 3 ? (4.0 * std::ldexp(1.0, -22) + std::ldexp(1.0, -21) * sq)
                                 : (std::ldexp(1.0, -10) * 1.001 + std::ldexp(1.0, -22) * sq);
  const double accum = (terms * dd + 64.0) * u23 * 1.01;
  *c1 = static_cast<float>(2.0 * (prod + accum));
  *c2 = static_cast<float>((dd + 4.0) * u23);
}

// host copy of an offsets array (device or host input), validated
int host_offsets(bvss_index* idx, const int64_t* qoff_in, int64_t nq, bool dev_ptrs, std::vector<int64_t>& out) {
  out.resize(nq + 1);
  if (dev_ptrs) {
    BVSS_CUDA(cudaMemcpyAsync(out.data(), qoff_in, (nq + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, idx->stream));
    BVSS_CUDA(cudaStreamSynchronize(idx->stream));
  } else {
    std::memcpy(out.data(), qoff_in, (nq + 1) * sizeof(int64_t));
  }
  return check_offsets(out.data(), nq, "query");
}

// ---- query preparation (a-4, Alg 6 lines 1-2): copy, encode (+norms, fp16 split), sketch.
// `queries` points at row qoff_host[0] == 0 of this batch; qoff_host is validated.
int prepare_queries(bvss_index* idx, bvss_search_ctx* c, const float* queries, const std::vector<int64_t>& qoff_host,
                    bool vec_dev, bool validate) {
  const int64_t nq = static_cast<int64_t>(qoff_host.size()) - 1;
  c->nq = nq;
  c->qoff_host = qoff_host;
  c->nqvec = qoff_host[nq];
  int max_mq = 0;
  for (int64_t i = 0; i < nq; ++i) {
    const int64_t sz = qoff_host[i + 1] - qoff_host[i];
    if (sz > max_mq) max_mq = static_cast<int>(sz > (1 << 30) ? (1 << 30) : sz);
  }
  c->max_mq = max_mq;
  if (max_mq > 256) BVSS_FAIL(BVSS_EUNSUPPORTED, "query sets of more than 256 vectors are not supported in this build");
  const int d = idx->d, dpad = idx->dpad, R = idx->m / 32;
  // refine operand rows: every query starts on an 8-aligned row (SW128 swizzle phase), +slack for
  // the N = ceil(m_q/16)*16 rows a tile reads
  std::vector<int64_t> qrow_h(nq), dst_h(c->nqvec);
  int64_t run = 0;
  for (int64_t i = 0; i < nq; ++i) {
    qrow_h[i] = run;
    for (int64_t v = qoff_host[i]; v < qoff_host[i + 1]; ++v) dst_h[v] = run + (v - qoff_host[i]);
    run += (qoff_host[i + 1] - qoff_host[i] + 7) & ~int64_t(7);
  }
  c->qrows = run + 256;
  cudaEventRecord(idx->ev[0], idx->stream);
  BVSS_TRY(c->alloc(c->nqvec * d * sizeof(float), reinterpret_cast<void**>(&c->qv)));
  BVSS_TRY(c->alloc((nq + 1) * sizeof(int64_t), reinterpret_cast<void**>(&c->qoff)));
  BVSS_TRY(c->alloc(c->nqvec * sizeof(float), reinterpret_cast<void**>(&c->qnorm)));
  BVSS_TRY(c->alloc(c->qrows * dpad * sizeof(__half), reinterpret_cast<void**>(&c->qhi)));
  BVSS_TRY(c->alloc(c->qrows * dpad * sizeof(__half), reinterpret_cast<void**>(&c->qlo)));
  BVSS_TRY(c->alloc(c->qrows * sizeof(float), reinterpret_cast<void**>(&c->qscale)));
  BVSS_TRY(c->alloc(nq * sizeof(int64_t), reinterpret_cast<void**>(&c->qrow)));
  int64_t* dst_row;
  BVSS_TRY(c->alloc(c->nqvec * sizeof(int64_t), reinterpret_cast<void**>(&dst_row)));
  BVSS_CUDA(cudaMemcpyAsync(c->qrow, qrow_h.data(), nq * sizeof(int64_t), cudaMemcpyHostToDevice, idx->stream));
  BVSS_CUDA(cudaMemcpyAsync(dst_row, dst_h.data(), c->nqvec * sizeof(int64_t), cudaMemcpyHostToDevice, idx->stream));
  BVSS_TRY(to_device(idx, c->qv, queries, c->nqvec * d * sizeof(float), vec_dev));
  BVSS_CUDA(cudaMemcpyAsync(c->qoff, c->qoff_host.data(), (nq + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, idx->stream));
  if (validate) {
    int* bad;
    BVSS_TRY(c->alloc(sizeof(int), reinterpret_cast<void**>(&bad)));
    BVSS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), idx->stream));
    BVSS_TRY(launch_finite_check(c->qv, c->nqvec * d, bad, idx->num_sms, idx->stream));
    int hbad = 0;
    BVSS_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, idx->stream));
    BVSS_CUDA(cudaStreamSynchronize(idx->stream));
    if (hbad) BVSS_FAIL(BVSS_ENONFINITE, "queries contain NaN or Inf");
  }
  BVSS_TRY(c->alloc(c->nqvec * R * sizeof(uint32_t), reinterpret_cast<void**>(&c->qcodes)));
  cudaEventRecord(idx->ev[1], idx->stream);
  BVSS_TRY(launch_encode(c->qv, c->nqvec, d, idx->Wt, idx->m, idx->s, idx->L, c->qcodes, c->qnorm, c->qhi, c->qlo, c->qscale,
                         dpad, c->qrows, dst_row, refine_kcs(dpad), idx->num_sms, idx->stream));
  const int cps = chunks_per_set(idx);
  BVSS_TRY(c->alloc(nq * cps * 16, &c->qsk));
  BVSS_TRY(c->alloc(nq * sizeof(int32_t), reinterpret_cast<void**>(&c->qmass)));
  BVSS_TRY(launch_sketch(c->qcodes, idx->m, c->qoff, nq, idx->sketch, c->qsk, c->qmass, 1, cps, idx->num_sms,
                         idx->stream));
  if (idx->score == 1) {  // OVERLAP (R24): key = K0 + 0 - 2 <S_Q, S_i> with zero database masses (build)
    fill_i32_kernel<<<static_cast<int>((nq + 255) / 256), 256, 0, idx->stream>>>(c->qmass, nq,
                                                                              static_cast<int32_t>(overlap_k0(idx)));
    idx->stats.kernel_launches += 1;
    BVSS_TRY(post_launch("fill_i32_kernel", idx->stream));
  }
  if (gated(idx)) {  // stage 1 (Alg 6 lines 1, 3-4): the top-A positions of every query's count Bloom filter
    BVSS_TRY(c->alloc(static_cast<size_t>(nq) * idx->gate_A * 4, reinterpret_cast<void**>(&c->gate_pos)));
    BVSS_TRY(launch_gate_positions(c->qcodes, c->qoff, static_cast<int>(nq), static_cast<int>(idx->m),
                                   static_cast<int>(idx->gate_A), c->gate_pos, idx->stream));
    idx->stats.kernel_launches += 1;
  }
  cudaEventRecord(idx->ev[2], idx->stream);
  idx->stats.kernel_launches += 2;
  return BVSS_OK;
}

bool use_tc_scan(const bvss_index* idx) {
  static const bool simt = getenv("BVSS_SCAN_SIMT") != nullptr;  // developer switch: SIMT popc/dp4a scan
  if (idx->score == 3 && idx->sketch == BVSS_SKETCH_COUNT_U8) return false;  // L1 (R26): no GEMM form
  return idx->m % (idx->sketch == BVSS_SKETCH_BINARY ? 256 : 128) == 0 && !simt;
}
// the SIMT scan's kind: the sketch kind, or 2 = count sketches scored L1 (R26)
int scan_kind(const bvss_index* idx) {
  return (idx->score == 3 && idx->sketch == BVSS_SKETCH_COUNT_U8) ? 2 : static_cast<int>(idx->sketch);
}
// database operand of the tensor-core scan (binary: FP4 expansion; count: the counters themselves)
const void* scan_operand(const bvss_index* idx, bool sample) {
  if (idx->sketch == BVSS_SKETCH_BINARY) return sample ? idx->smp_skx : idx->skx;
  return sample ? idx->smp_sk : idx->sk;
}

// tensor-core scan operands: queries expanded to [m/16][qpad][16 B] (scan_tc.cu)
int expand_alloc(bvss_index* idx, bvss_search_ctx* c) {
  c->qpad = static_cast<int>(ceil_div<int64_t>(c->nq, 128) * 128);
  return idx->ws.get("scan_qx", static_cast<size_t>(scan_tc_units(idx->sketch, idx->m)) * 16 * c->qpad, &c->qx);
}

int alloc_select_state(bvss_index* idx, bvss_search_ctx* c) {
  const int nq = static_cast<int>(c->nq);
  BVSS_TRY(c->alloc(nq * sizeof(uint32_t), reinterpret_cast<void**>(&c->sel.prefix)));
  BVSS_TRY(c->alloc(nq * sizeof(int64_t), reinterpret_cast<void**>(&c->sel.below)));
  BVSS_TRY(c->alloc(nq * sizeof(int64_t), reinterpret_cast<void**>(&c->sel.teff)));
  BVSS_TRY(c->alloc(nq * sizeof(int64_t), reinterpret_cast<void**>(&c->sel.eq)));
  BVSS_TRY(c->alloc(nq * sizeof(int64_t), reinterpret_cast<void**>(&c->sel.quota)));
  BVSS_TRY(c->alloc(nq * sizeof(int32_t), reinterpret_cast<void**>(&c->sel.digit)));
  BVSS_TRY(c->alloc(static_cast<size_t>(nq) * kHistBins * sizeof(int32_t), reinterpret_cast<void**>(&c->local_hist)));
  c->key_bits = key_bits_for(idx->filter == 1 ? static_cast<int>(BVSS_SKETCH_BINARY) : static_cast<int>(idx->sketch),
                             idx->m);  // (Alg 2: Haus^H <= m, like a binary Hamming score)
  if (gated(idx)) c->key_bits = 8 * key_size_of(idx);  // the gate's top bit
  if (idx->score == 1) {  // OVERLAP keys span [0, K0]
    c->key_bits = 1;
    while ((overlap_k0(idx) >> c->key_bits) != 0) ++c->key_bits;
  }
  c->rounds = rounds_for(c->key_bits);
  c->next_round = 0;
  return BVSS_OK;
}

// Key rows of queries [q0, q0 + ns) of a prepared batch over all n sets: the sketch scan (K3, tensor core or
// SIMT) or Alg 2's Haus^H over the per-vector codes (gate.cu), then the stage-1 gate's top bit on rejected sets.
int scan_keys(bvss_index* idx, bvss_search_ctx* c, int q0, int ns, void* keys, int64_t key_stride) {
  const int64_t n = idx->n;
  if (idx->filter == 1) {
    BVSS_TRY(launch_alg2_keys(c->qcodes, c->qoff + q0, ns, c->max_mq, idx->codes, idx->off, n, idx->m,
                              static_cast<uint16_t*>(keys), key_stride, idx->num_sms, idx->stream));
    idx->stats.kernel_launches += 1;
  } else {
    const int cps = chunks_per_set(idx);
    const void* sq = static_cast<const uint8_t*>(c->qsk) + static_cast<size_t>(q0) * cps * 16;
    if (use_tc_scan(idx)) {
      BVSS_TRY(expand_alloc(idx, c));
      int* wc;
      BVSS_TRY(idx->ws.get("scan_counter", sizeof(int), reinterpret_cast<void**>(&wc)));
      BVSS_TRY(launch_scan_tc(idx->sketch, scan_operand(idx, false), idx->mass, n, n, idx->m, sq, c->qmass + q0, ns,
                              c->qx, c->qpad, keys, key_stride, wc, idx->num_sms, idx->stream, nullptr, nullptr,
                              nullptr, nullptr, 0, 0, true));
      idx->stats.kernel_launches += 2;
      idx->stats.scan_bytes += scan_tc_db_bytes(idx->sketch, idx->m, n, ns, idx->num_sms);
    } else {
      BVSS_TRY(launch_scan(scan_kind(idx), idx->sk, idx->mass, n, n, idx->m, sq, c->qmass + q0, ns, keys, key_stride,
                           idx->num_sms, idx->stream));
      idx->stats.kernel_launches += 1;
      idx->stats.scan_bytes += static_cast<uint64_t>(ceil_div<int64_t>(ns, 8)) * n * chunks_per_set(idx) * 16;
    }
    idx->stats.scan_macs += static_cast<uint64_t>(ns) * n * idx->m;
  }
  if (gated(idx)) {
    BVSS_TRY(launch_gate_keys(key_size_of(idx), keys, key_stride, n, ns, c->gate_pos + static_cast<int64_t>(q0) * idx->gate_A,
                              static_cast<int>(idx->gate_A), idx->planes, idx->gW, idx->num_sms, idx->stream));
    idx->stats.kernel_launches += 1;
  }
  return BVSS_OK;
}

// full-key scan (every score written) + select state init; the caller drives the select rounds
int scan_batch(bvss_index* idx, bvss_search_ctx* c) {
  const int64_t n = idx->n;
  const int key_size = key_size_of(idx);
  c->key_stride = (n + 7) & ~int64_t(7);
  BVSS_TRY(idx->ws.get("keys", static_cast<size_t>(c->nq) * c->key_stride * key_size, &c->keys));
  BVSS_TRY(scan_keys(idx, c, 0, static_cast<int>(c->nq), c->keys, c->key_stride));
  cudaEventRecord(idx->ev[3], idx->stream);
  BVSS_TRY(alloc_select_state(idx, c));
  BVSS_TRY(launch_select_init(c->sel, static_cast<int>(c->nq), c->teff, idx->stream));
  return BVSS_OK;
}

bool sampled_select_eligible(const bvss_index* idx) {
  if (!use_tc_scan(idx) || idx->ns == 0 || gated(idx) || idx->filter == 1) return false;
  if (idx->select_mode == 2) return true;
  if (idx->select_mode == 1) return false;
  // auto: binary sketches only.  Count-sketch L2^2 keys of small sets tie massively (a singleton's key
  // depends only on its overlap with the query), so the emission buffers overflow at the threshold and
  // the batch would fall back anyway (measured on cfg4: every batch).
  return idx->n >= 65536 && idx->sketch == BVSS_SKETCH_BINARY;
}

// Sampled-threshold selection (select_mode 2) for one prepared batch: the
// k_s-th smallest key over the database sample estimates a per-query threshold
// tau_hat that lets ~k_s n / ns >= T keys through; the fused scan emits only keys
// <= tau_hat and select_buf_kernel picks the exact top-teff (key, id) from them.
// *ok = false when some query's buffer under- or overflowed (the caller then
// runs the full-key path for this batch).
int select_sampled(bvss_index* idx, bvss_search_ctx* c, bool* ok) {
  const int nq = static_cast<int>(c->nq);
  const int64_t n = idx->n, ns = idx->ns;
  const int key_size = key_size_of(idx);
  const double f = static_cast<double>(ns) / static_cast<double>(n);
  const double mu = static_cast<double>(c->teff) * f;
  int64_t ks = static_cast<int64_t>(std::ceil(mu + 5.0 * std::sqrt(mu) + 4.0));
  if (ks > ns) ks = ns;
  int64_t cap = static_cast<int64_t>(std::ceil(2.0 * static_cast<double>(ks) / f)) + 8192;
  if (cap < c->teff) cap = c->teff;
  if (cap > n) cap = n;
  if (const char* e = getenv("BVSS_DEBUG_EMIT_CAP")) cap = atoll(e);  // developer/test switch: force overflows
  cap = (cap + 7) & ~int64_t(7);
  BVSS_TRY(expand_alloc(idx, c));
  int* wc;
  BVSS_TRY(idx->ws.get("scan_counter", sizeof(int), reinterpret_cast<void**>(&wc)));
  // 1. scan the sample, full keys
  const int64_t sstride = (ns + 7) & ~int64_t(7);
  void* skeys;
  BVSS_TRY(idx->ws.get("sample_keys", static_cast<size_t>(nq) * sstride * key_size, &skeys));
  BVSS_TRY(launch_scan_tc(idx->sketch, scan_operand(idx, true), idx->smp_mass, ns, ns, idx->m, c->qsk, c->qmass, nq, c->qx,
                          c->qpad, skeys, sstride, wc, idx->num_sms, idx->stream, nullptr, nullptr, nullptr, nullptr, 0,
                          0, true));
  // 2. tau_hat = k_s-th smallest sample key (exact radix select on the sample)
  BVSS_TRY(alloc_select_state(idx, c));
  BVSS_TRY(launch_select_init(c->sel, nq, ks, idx->stream));
  for (int r = 0; r < c->rounds; ++r) {
    BVSS_TRY(launch_select_hist(key_size, skeys, sstride, ns, nq, c->sel, c->key_bits, r, c->local_hist, idx->stream));
    BVSS_TRY(launch_select_resolve(c->local_hist, c->sel, nq, c->key_bits, r, idx->stream));
  }
  // 3. fused scan: emit (id, key) with key <= tau_hat
  int32_t *cnt, *bid;
  uint32_t* bkey;
  BVSS_TRY(idx->ws.get("emit_cnt", nq * sizeof(int32_t), reinterpret_cast<void**>(&cnt)));
  BVSS_TRY(idx->ws.get("emit_id", static_cast<size_t>(nq) * cap * 4, reinterpret_cast<void**>(&bid)));
  BVSS_TRY(idx->ws.get("emit_key", static_cast<size_t>(nq) * cap * 4, reinterpret_cast<void**>(&bkey)));
  BVSS_CUDA(cudaMemsetAsync(cnt, 0, nq * sizeof(int32_t), idx->stream));
  BVSS_TRY(launch_scan_tc(idx->sketch, scan_operand(idx, false), idx->mass, n, n, idx->m, c->qsk, c->qmass, nq, c->qx, c->qpad, nullptr,
                          0, wc, idx->num_sms, idx->stream, c->sel.prefix, cnt, bid, bkey, static_cast<int>(cap),
                          c->id_base, false));
  idx->stats.scan_bytes += scan_tc_db_bytes(idx->sketch, idx->m, n, nq, idx->num_sms) +
                           scan_tc_db_bytes(idx->sketch, idx->m, ns, nq, idx->num_sms);
  idx->stats.scan_macs += static_cast<uint64_t>(nq) * (n + ns) * idx->m;
  cudaEventRecord(idx->ev[3], idx->stream);
  // 4. exact top-teff from the buffers
  BVSS_TRY(c->alloc(static_cast<size_t>(nq) * c->T * sizeof(int32_t), reinterpret_cast<void**>(&c->cand)));
  BVSS_TRY(c->alloc(nq * sizeof(int32_t), reinterpret_cast<void**>(&c->count)));
  int* fail;
  BVSS_TRY(idx->ws.get("select_fail", sizeof(int), reinterpret_cast<void**>(&fail)));
  BVSS_CUDA(cudaMemsetAsync(fail, 0, sizeof(int), idx->stream));
  BVSS_TRY(launch_select_buf(cnt, bkey, bid, static_cast<int>(cap), static_cast<int>(c->teff), c->key_bits, c->T, nq,
                             c->cand, c->count, fail, idx->stream));
  c->cand_sorted = select_buf_sorted(static_cast<int>(c->teff));
  cudaEventRecord(idx->ev[4], idx->stream);
  idx->stats.kernel_launches += 4 + 2 * c->rounds;
  int hf = 0;
  BVSS_CUDA(cudaMemcpyAsync(&hf, fail, sizeof(int), cudaMemcpyDeviceToHost, idx->stream));
  BVSS_CUDA(cudaStreamSynchronize(idx->stream));
  *ok = hf == 0;
  idx->stats.select_batches += 1;
  if (!*ok) idx->stats.select_fallbacks += 1;
  return BVSS_OK;
}

int emit_candidates(bvss_index* idx, bvss_search_ctx* c) {
  const int nq = static_cast<int>(c->nq);
  const int key_size = key_size_of(idx);
  BVSS_TRY(c->alloc(static_cast<size_t>(nq) * c->T * sizeof(int32_t), reinterpret_cast<void**>(&c->cand)));
  BVSS_TRY(c->alloc(nq * sizeof(int32_t), reinterpret_cast<void**>(&c->count)));
  BVSS_TRY(launch_select_emit(key_size, c->keys, c->key_stride, idx->n, nq, c->sel, c->T, c->id_base, c->cand, nullptr,
                              c->count, idx->stream, key_limit_of(idx)));
  cudaEventRecord(idx->ev[4], idx->stream);
  idx->stats.kernel_launches += 1;
  return BVSS_OK;
}

// Full-key candidate selection for a prepared batch, in sub-batches whose key rows fit 4 GB: the
// fallback of the sampled-threshold path (same result, more memory traffic).
int fallback_full(bvss_index* idx, bvss_search_ctx* c) {
  const int nq = static_cast<int>(c->nq);
  const int64_t n = idx->n;
  const int key_size = key_size_of(idx);
  const int64_t key_stride = (n + 7) & ~int64_t(7);
  double sub_bytes = 4.0 * (1ull << 30);
  if (const char* e = getenv("BVSS_DEBUG_SUBBATCH_BYTES")) sub_bytes = atof(e);  // test switch: many sub-batches
  int64_t sub = static_cast<int64_t>(sub_bytes / (static_cast<double>(key_stride) * key_size));
  if (sub < 1) sub = 1;
  if (sub > nq) sub = nq;
  void* keys;
  BVSS_TRY(idx->ws.get("keys", static_cast<size_t>(sub) * key_stride * key_size, &keys));
  BVSS_TRY(alloc_select_state(idx, c));
  BVSS_TRY(c->alloc(static_cast<size_t>(nq) * c->T * sizeof(int32_t), reinterpret_cast<void**>(&c->cand)));
  BVSS_TRY(c->alloc(nq * sizeof(int32_t), reinterpret_cast<void**>(&c->count)));
  for (int q0 = 0; q0 < nq; q0 += static_cast<int>(sub)) {
    const int ns = static_cast<int>(q0 + sub <= nq ? sub : nq - q0);
    BVSS_TRY(scan_keys(idx, c, q0, ns, keys, key_stride));
    SelectState s2 = c->sel;
    s2.prefix += q0;
    s2.below += q0;
    s2.teff += q0;
    s2.eq += q0;
    s2.quota += q0;
    s2.digit += q0;
    BVSS_TRY(launch_select_init(s2, ns, c->teff, idx->stream));
    for (int r = 0; r < c->rounds; ++r) {
      BVSS_TRY(launch_select_hist(key_size, keys, key_stride, n, ns, s2, c->key_bits, r, c->local_hist, idx->stream));
      BVSS_TRY(launch_select_resolve(c->local_hist, s2, ns, c->key_bits, r, idx->stream));
    }
    BVSS_TRY(launch_select_emit(key_size, keys, key_stride, n, ns, s2, c->T, c->id_base,
                                c->cand + static_cast<int64_t>(q0) * c->T, nullptr, c->count + q0, idx->stream,
                                key_limit_of(idx)));
    idx->stats.kernel_launches += 4 + 2 * c->rounds;
  }
  cudaEventRecord(idx->ev[4], idx->stream);
  c->cand_sorted = true;  // order-preserving emission
  return BVSS_OK;
}

// refine + top-k over c->cand / c->count
int refine_topk(bvss_index* idx, bvss_search_ctx* c, int64_t* out_ids_dev, float* out_dist_dev) {
  const int nq = static_cast<int>(c->nq);
  int exact_all = 0;
  float c1, c2;
  error_consts(idx, &c1, &c2);
  if (idx->terms != 0) {  // tensor path (query sets > 128 rows: per query on the exact path, refine.cu)
    if (!c->approx)  // once per context (brute force calls this per chunk)
      BVSS_TRY(c->alloc(static_cast<size_t>(nq) * c->T * sizeof(float), reinterpret_cast<void**>(&c->approx)));
    if (idx->metric == 1 && !c->approx_err)
      BVSS_TRY(c->alloc(static_cast<size_t>(nq) * c->T * sizeof(float), reinterpret_cast<void**>(&c->approx_err)));
    int* counter;
    BVSS_TRY(idx->ws.get("work_counter", sizeof(int), reinterpret_cast<void**>(&counter)));
    unsigned long long* rows;
    BVSS_TRY(idx->ws.get("rows_counter", sizeof(unsigned long long), reinterpret_cast<void**>(&rows)));
    int32_t* bounds = nullptr;  // range bounds of the range-major refine (refine.cu)
    {
      const int64_t rs = refine_range_sets(idx->n, idx->prows, idx->dpad, c->T);
      if (rs > 0 && c->cand_sorted) {
        const int64_t nr = (idx->n + rs - 1) / rs;
        const size_t bb = ((static_cast<size_t>(nq) * (nr + 1) * 4) + 15) & ~size_t(15);
        BVSS_TRY(idx->ws.get("refine_bounds", bb + static_cast<size_t>(nq) * (16 + 32 * 8),
                             reinterpret_cast<void**>(&bounds)));
      }
    }
    BVSS_TRY(launch_refine_tc(idx->hi, idx->lo, idx->vscale, idx->prows, idx->pbase, idx->vnorm, idx->off, idx->dpad, c->qhi,
                              c->qlo, c->qscale, c->qrows,
                              c->qrow, c->qnorm, c->qoff, c->max_mq, c->cand, c->count, c->T, nq, c->id_base,
                              c->approx, idx->terms, counter, rows, idx->num_sms, c->cand_sorted ? idx->n : 0, bounds,
                              idx->metric, c->approx_err, c1, c2, idx->vmax2, idx->stream));
    idx->stats.kernel_launches += 1;
  } else {
    exact_all = 1;
  }
  cudaEventRecord(idx->ev[5], idx->stream);
  int64_t* fix;
  BVSS_TRY(idx->ws.get("fixup_counter", sizeof(int64_t), reinterpret_cast<void**>(&fix)));
  BVSS_CUDA(cudaMemsetAsync(fix, 0, sizeof(int64_t), idx->stream));
  void* scratch;
  BVSS_TRY(idx->ws.get("topk_scratch", static_cast<size_t>(nq) * c->T * 8, &scratch));
  BVSS_TRY(launch_topk_fixup(c->approx, c->cand, c->count, c->T, c->k, idx->V, idx->off, c->id_base, idx->d, c->qv,
                             c->qoff, c->qnorm, idx->vmax2, c1, c2, exact_all, out_ids_dev, out_dist_dev, nq, fix,
                             scratch, idx->metric, c->approx_err, idx->max_rows, c->max_mq, idx->stream));
  cudaEventRecord(idx->ev[6], idx->stream);
  idx->stats.kernel_launches += 1;
  return BVSS_OK;
}

float ev_ms(bvss_index* idx, int a, int b);

// ------------------------------------------------ dense (candidate-major) refine, dense.cu --
// The database operand of the dense kernel (fp16 x / S, S a power of two >= max|x|) and its tile plan (runs
// of whole consecutive sets of <= 144 rows; larger sets go to the exact path), built on first use.
int ensure_dense(bvss_index* idx) {
  if (idx->hd) return BVSS_OK;
  if (idx->dpad > dense_max_dpad()) BVSS_FAIL(BVSS_EUNSUPPORTED, "dense refine needs d <= %d", dense_max_dpad());
  const float mx = std::sqrt(idx->vmax2);  // max |x_i| <= max |x|
  int ex = 0;
  if (mx > 0.0f) std::frexp(mx, &ex);      // mx = f 2^ex, f in [0.5, 1): 2^ex > mx
  idx->dense_s = std::ldexp(1.0f, ex);
  const size_t hb = static_cast<size_t>(idx->nvec) * idx->dpad * 2;
  BVSS_CUDA(cudaMalloc(reinterpret_cast<void**>(&idx->hd), hb));
  idx->owned_bytes += hb;
  BVSS_TRY(launch_dense_db_operand(idx->V, idx->nvec, idx->d, idx->dpad, 1.0f / idx->dense_s, idx->hd, idx->num_sms,
                                   idx->stream));
  const size_t vb = static_cast<size_t>(idx->nvec) * 32;
  BVSS_CUDA(cudaMalloc(reinterpret_cast<void**>(&idx->va), vb));
  idx->owned_bytes += vb;
  BVSS_TRY(launch_dense_norm_operand(idx->vnorm, idx->nvec, 1.0f / (idx->dense_s * idx->dense_s), idx->va,
                                     idx->num_sms, idx->stream));
  std::vector<int32_t> s0, s1, huge;
  const std::vector<int64_t>& o = idx->off_h;
  const int64_t cap_rows = dense_tile_rows();  // dense.cu kDenseN
  for (int64_t i = 0; i < idx->n;) {
    if (o[i + 1] - o[i] > cap_rows) {
      huge.push_back(static_cast<int32_t>(i));
      ++i;
      continue;
    }
    const int64_t start = i;
    while (i < idx->n && o[i + 1] - o[i] <= cap_rows && o[i + 1] - o[start] <= cap_rows) ++i;
    s0.push_back(static_cast<int32_t>(start));
    s1.push_back(static_cast<int32_t>(i));
  }
  idx->dntiles = static_cast<int>(s0.size());
  idx->dnhuge = static_cast<int>(huge.size());
  const size_t tb = std::max<size_t>(s0.size(), 1) * 4;
  BVSS_CUDA(cudaMalloc(reinterpret_cast<void**>(&idx->dtile_s0), tb));
  BVSS_CUDA(cudaMalloc(reinterpret_cast<void**>(&idx->dtile_s1), tb));
  BVSS_CUDA(cudaMalloc(reinterpret_cast<void**>(&idx->dhuge), std::max<size_t>(huge.size(), 1) * 4));
  idx->owned_bytes += 2 * tb;
  if (!s0.empty()) {
    BVSS_CUDA(cudaMemcpyAsync(idx->dtile_s0, s0.data(), s0.size() * 4, cudaMemcpyHostToDevice, idx->stream));
    BVSS_CUDA(cudaMemcpyAsync(idx->dtile_s1, s1.data(), s1.size() * 4, cudaMemcpyHostToDevice, idx->stream));
  }
  if (!huge.empty())
    BVSS_CUDA(cudaMemcpyAsync(idx->dhuge, huge.data(), huge.size() * 4, cudaMemcpyHostToDevice, idx->stream));
  BVSS_CUDA(cudaStreamSynchronize(idx->stream));  // host vectors go out of scope
  idx->dtile_s0_h = s0;
  return BVSS_OK;
}

// the dense path takes a batch when every query set fits one 32-lane warp of the query tile, the metric is
// Hausdorff and d fits the resident query tile
bool dense_supported(const bvss_index* idx, const bvss_search_ctx* c) {
  return idx->metric == 0 && idx->terms != 0 && idx->dpad <= dense_max_dpad() && c->max_mq <= 32 && c->k <= 32;
}

// BVSS_DENSE: 0 = never, 1 = whenever supported, unset = auto (the candidate budget is a large fraction of
// the database: gathering T candidates per query then costs more than one dense pass)
bool dense_wanted(const bvss_index* idx, int64_t teff) {
  static const int env = [] {
    const char* e = getenv("BVSS_DENSE");
    return e ? atoi(e) : -1;
  }();
  if (env == 0 || idx->metric != 0 || idx->terms == 0 || idx->dpad > dense_max_dpad()) return false;
  if (env == 1) return true;
  return teff * 8 >= idx->n;
}

// Exact top-k of a prepared batch by the dense kernel: every (query, set) Gram on the tensor cores, the
// branch-and-bound prune, the emitted candidate lists, then K6 (topk_exact_kernel) on those lists.
// mask: optional candidate bitmap (row q at mask + q * mask_stride); ntiles_use: dense tiles to scan (a
// prefix, for brute force over the first set_limit sets; -1 = all).  *done = false when the batch is not supported or a
// candidate list overflowed (the caller then runs the query-major path; the result is the same).
int dense_refine_topk(bvss_index* idx, bvss_search_ctx* c, const uint32_t* mask, int64_t mask_stride, int ntiles_use,
                      int64_t* out_ids_dev, float* out_dist_dev, bool* done) {
  *done = false;
  if (!dense_supported(idx, c)) return BVSS_OK;
  BVSS_TRY(ensure_dense(idx));
  if (ntiles_use < 0 || ntiles_use > idx->dntiles) ntiles_use = idx->dntiles;  // (-1: every tile)
  const int nq = static_cast<int>(c->nq), k = c->k;
  // query packing: best fit (decreasing sizes) into 32-row warp bins, 4 bins per 128-row tile
  std::vector<int> order(nq);
  for (int q = 0; q < nq; ++q) order[q] = q;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return c->qoff_host[a + 1] - c->qoff_host[a] > c->qoff_host[b + 1] - c->qoff_host[b];
  });
  std::vector<std::vector<int>> by_space(33);
  std::vector<int> fill;
  std::vector<std::vector<int>> bins;
  for (int q : order) {
    const int m = static_cast<int>(c->qoff_host[q + 1] - c->qoff_host[q]);
    int b = -1;
    for (int sp = m; sp <= 32 && b < 0; ++sp)
      if (!by_space[sp].empty()) {
        b = by_space[sp].back();
        by_space[sp].pop_back();
      }
    if (b < 0) {
      b = static_cast<int>(bins.size());
      bins.emplace_back();
      fill.push_back(0);
    }
    bins[b].push_back(q);
    fill[b] += m;
    by_space[32 - fill[b]].push_back(b);
  }
  const int ntq = static_cast<int>(((bins.size() + 3) / 4 + 1) & ~size_t(1));  // (the kernel pairs query tiles)
  const int64_t rows = static_cast<int64_t>(ntq) * 128;
  std::vector<int32_t> rowmap(rows, -1), rowq(rows, -1);
  for (size_t b = 0; b < bins.size(); ++b) {
    int64_t r = static_cast<int64_t>(b) * 32;  // tile b/4, lane quarter b%4
    for (int q : bins[b])
      for (int64_t v = c->qoff_host[q]; v < c->qoff_host[q + 1]; ++v, ++r) {
        rowmap[r] = static_cast<int32_t>(v);
        rowq[r] = q;
      }
  }
  const int ntiles = ntiles_use;
  // work units = (query tile pair, database range).  Dynamic schedule (default): ranges of kDenseTPR tiles
  // handed out range-major by a global counter (all pairs stream the same ranges at once: L2 reuse; tau of
  // a unit starts from the query's lists of the ranges before it).  Static (BVSS_DENSE_DYN=0): at least two
  // units per SM pair, pair-major.
  int dyn = 1;
  if (const char* e = getenv("BVSS_DENSE_DYN")) dyn = atoi(e) != 0;
  int tpr = 256;
  if (const char* e = getenv("BVSS_DENSE_TPR")) tpr = atoi(e) > 0 ? atoi(e) : tpr;  // developer switch
  int R = dyn ? static_cast<int>(ceil_div<int64_t>(ntiles, tpr))
              : static_cast<int>(ceil_div<int64_t>(2 * idx->num_sms, ntq));
  if (!dyn && R < 4) R = 4;
  if (const char* e = getenv("BVSS_DENSE_R")) R = atoi(e) > 0 ? atoi(e) : R;  // developer switch: database ranges
  if (R > ntiles) R = ntiles < 1 ? 1 : ntiles;
  if (static_cast<int64_t>(ntq / 2) * R >= (int64_t(1) << 31)) R = static_cast<int>((int64_t(1) << 30) / (ntq / 2));
  // (dyn: a unit's tau starts from the lists of the ranges run before it, so the emissions per query grow
  // like those of a few ranges, not of R)
  const int R_emit = dyn ? std::min(R, 8) : R;
  const double spl = std::max(1.0, static_cast<double>(idx->n) / (static_cast<double>(R_emit) * dense_epi_sub() * k));
  const double lists_pq = static_cast<double>(R_emit) * dense_epi_sub();  // bound lists per query
  int64_t cap = static_cast<int64_t>(lists_pq * k * (2.0 + std::log(spl)) * 2.0) + idx->dnhuge + 1024;
  cap = (cap + 255) & ~int64_t(255);
  if (const char* e = getenv("BVSS_DEBUG_DENSE_CAP")) cap = atoll(e);  // test switch: force overflows (cap < k)
  // query max norm -> S_q
  unsigned int* vmax;
  BVSS_TRY(idx->ws.get("vmax", sizeof(unsigned int), reinterpret_cast<void**>(&vmax)));
  BVSS_CUDA(cudaMemsetAsync(vmax, 0, sizeof(unsigned int), idx->stream));
  max_float_kernel<<<idx->num_sms, 256, 0, idx->stream>>>(c->qnorm, c->nqvec, vmax);
  BVSS_TRY(post_launch("max_float_kernel", idx->stream));
  unsigned int hv = 0;
  BVSS_CUDA(cudaMemcpyAsync(&hv, vmax, sizeof(hv), cudaMemcpyDeviceToHost, idx->stream));
  BVSS_CUDA(cudaStreamSynchronize(idx->stream));
  float qmax2;
  std::memcpy(&qmax2, &hv, 4);
  int ex = 0;
  if (qmax2 > 0.0f) std::frexp(std::sqrt(qmax2), &ex);
  const float sq = std::ldexp(1.0f, ex);
  // the norm chunk of the query tile: (alpha, alpha, 0 ...) on every row, alpha = -S_db / (2 S_q) (a power of
  // two; it must be a normal fp16 number for the product to stay exact)
  const float alpha = -idx->dense_s / (2.0f * sq);
  if (std::fabs(alpha) < std::ldexp(1.0f, -14) || std::fabs(alpha) > 32768.0f) return BVSS_OK;  // (query-major)
  std::vector<__half> qa_h(128 * 16, __float2half_rn(0.0f));
  for (int r = 0; r < 128; ++r) qa_h[r * 16] = qa_h[r * 16 + 1] = __float2half_rn(alpha);
  // buffers
  __half *qd, *qa;
  int32_t *d_rowmap, *d_rowq, *lane_qid, *cnt, *ids;
  float *lane_qn, *qE, *tau0, *lists, *vals;
  unsigned long long* stat;
  const int64_t nlist = static_cast<int64_t>(nq) * R * dense_epi_sub() * k;
  BVSS_TRY(c->alloc(rows * idx->dpad * 2, reinterpret_cast<void**>(&qd)));
  BVSS_TRY(c->alloc(128 * 16 * 2, reinterpret_cast<void**>(&qa)));
  BVSS_CUDA(cudaMemcpyAsync(qa, qa_h.data(), 128 * 16 * 2, cudaMemcpyHostToDevice, idx->stream));
  BVSS_TRY(c->alloc(rows * 4, reinterpret_cast<void**>(&d_rowmap)));
  BVSS_TRY(c->alloc(rows * 4, reinterpret_cast<void**>(&d_rowq)));
  BVSS_TRY(c->alloc(rows * 4, reinterpret_cast<void**>(&lane_qid)));
  BVSS_TRY(c->alloc(rows * 4, reinterpret_cast<void**>(&lane_qn)));
  BVSS_TRY(c->alloc(nq * 4, reinterpret_cast<void**>(&qE)));
  BVSS_TRY(c->alloc(nq * 4, reinterpret_cast<void**>(&tau0)));
  BVSS_TRY(c->alloc(nlist * 4, reinterpret_cast<void**>(&lists)));
  BVSS_TRY(c->alloc(nq * 4, reinterpret_cast<void**>(&cnt)));
  BVSS_TRY(c->alloc(static_cast<size_t>(nq) * cap * 4, reinterpret_cast<void**>(&ids)));
  BVSS_TRY(c->alloc(static_cast<size_t>(nq) * cap * 4, reinterpret_cast<void**>(&vals)));
  BVSS_TRY(c->alloc(2 * sizeof(unsigned long long), reinterpret_cast<void**>(&stat)));
  int* unit_ctr;
  BVSS_TRY(c->alloc(sizeof(int), reinterpret_cast<void**>(&unit_ctr)));
  int* udone;
  BVSS_TRY(c->alloc(static_cast<size_t>(ntq / 2) * R * sizeof(int), reinterpret_cast<void**>(&udone)));
  BVSS_CUDA(cudaMemcpyAsync(d_rowmap, rowmap.data(), rows * 4, cudaMemcpyHostToDevice, idx->stream));
  BVSS_CUDA(cudaMemcpyAsync(d_rowq, rowq.data(), rows * 4, cudaMemcpyHostToDevice, idx->stream));
  BVSS_CUDA(cudaMemsetAsync(stat, 0, 2 * sizeof(unsigned long long), idx->stream));
  BVSS_TRY(launch_dense_query_operand(c->qv, c->qnorm, d_rowmap, d_rowq, rows, idx->d, idx->dpad, 1.0f / sq, qd,
                                      lane_qid, lane_qn, idx->num_sms, idx->stream));
  float c1, c2;
  error_consts(idx, &c1, &c2);
  // the accumulator also carries alpha (h + l) ~ |v|^2 / (2 S_q S_db): its fp32 accumulation adds at most
  // (dpad + 80) 2^-23 |v|^2 after the kappa scaling, and the (h, l) split 2^-21 |v|^2
  c2 += static_cast<float>((idx->dpad + 80.0) * std::ldexp(1.0, -23) * 1.01 + std::ldexp(1.0, -21));
  fill_f32_inf(tau0, nq, idx->stream);
  BVSS_TRY(launch_dense_prep(c->qoff, c->qnorm, nq, c1, c2, idx->vmax2, qE, lists, nlist, cnt, idx->dhuge,
                             idx->dnhuge, mask, mask_stride, c->id_base, ids, vals, static_cast<int>(cap),
                             idx->num_sms, idx->stream));
  cudaEventRecord(idx->ev[4], idx->stream);
  BVSS_TRY(launch_dense_hausdorff(qd, ntq, idx->hd, idx->nvec, idx->dpad, ntiles, idx->dtile_s0, idx->dtile_s1,
                                  idx->off, idx->va, qa, lane_qid, lane_qn, qE, tau0, -2.0f * sq * idx->dense_s, alpha,
                                  k, R,
                                  lists, cnt, ids, vals, static_cast<int>(cap), mask, mask_stride, c->id_base, stat,
                                  dyn, unit_ctr, udone, idx->num_sms, idx->stream));
  cudaEventRecord(idx->ev[5], idx->stream);
  idx->stats.kernel_launches += 6;
  // overflow check
  std::vector<int32_t> hc(nq);
  BVSS_CUDA(cudaMemcpyAsync(hc.data(), cnt, nq * 4, cudaMemcpyDeviceToHost, idx->stream));
  BVSS_CUDA(cudaMemcpyAsync(idx->dense_stat, stat, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            idx->stream));
  BVSS_CUDA(cudaStreamSynchronize(idx->stream));
  idx->stats.ms_refine += ev_ms(idx, 4, 5);  // (bvss_search rewrites it from its own event sums)
  for (int q = 0; q < nq; ++q)
    if (hc[q] > cap) {
      idx->stats.select_fallbacks += 1;  // (reported as a fallback of the dense path)
      return BVSS_OK;                    // *done stays false: the caller takes the query-major path
    }
  int64_t* fix;
  BVSS_TRY(idx->ws.get("fixup_counter", sizeof(int64_t), reinterpret_cast<void**>(&fix)));
  BVSS_CUDA(cudaMemsetAsync(fix, 0, sizeof(int64_t), idx->stream));
  void* scratch;
  BVSS_TRY(idx->ws.get("topk_scratch", static_cast<size_t>(nq) * cap * 8, &scratch));
  BVSS_TRY(launch_topk_fixup(vals, ids, cnt, static_cast<int>(cap), k, idx->V, idx->off, c->id_base, idx->d, c->qv,
                             c->qoff, c->qnorm, idx->vmax2, c1, c2, 0, out_ids_dev, out_dist_dev, nq, fix, scratch, 0,
                             nullptr, idx->max_rows, c->max_mq, idx->stream));
  cudaEventRecord(idx->ev[6], idx->stream);
  idx->stats.kernel_launches += 1;
  idx->stats.dense_batches += 1;
  idx->stats.dense_survivors += idx->dense_stat[0];
  idx->stats.dense_emitted += idx->dense_stat[1];
  idx->stats.dense_pairs += static_cast<uint64_t>(c->nqvec) * static_cast<uint64_t>(
      ntiles_use >= idx->dntiles ? idx->nvec : idx->off_h[idx->dtile_s0_h[ntiles_use]]);
  idx->stats.dense_flop += 2.0 * static_cast<double>(rows) * idx->dpad *
                           static_cast<double>(ntiles_use) * dense_tile_rows();
  *done = true;
  return BVSS_OK;
}

// candidate bitmap of a prepared batch (bit i of row q = set i is in the query's top-T): full-key scans and
// radix selects in sub-batches whose key rows fit 4 GB, written by select_bitmap_kernel
int dense_mask(bvss_index* idx, bvss_search_ctx* c, uint32_t** mask, int64_t* stride) {
  const int nq = static_cast<int>(c->nq);
  const int64_t n = idx->n;
  const int key_size = key_size_of(idx);
  const int64_t key_stride = (n + 7) & ~int64_t(7);
  double sub_bytes = 4.0 * (1ull << 30);
  if (const char* e = getenv("BVSS_DEBUG_SUBBATCH_BYTES")) sub_bytes = atof(e);
  int64_t sub = static_cast<int64_t>(sub_bytes / (static_cast<double>(key_stride) * key_size));
  if (sub < 1) sub = 1;
  if (sub > nq) sub = nq;
  const int64_t words = (n + 31) / 32;
  BVSS_TRY(c->alloc(static_cast<size_t>(nq) * words * 4, reinterpret_cast<void**>(mask)));
  BVSS_CUDA(cudaMemsetAsync(*mask, 0, static_cast<size_t>(nq) * words * 4, idx->stream));
  *stride = words;
  void* keys;
  BVSS_TRY(idx->ws.get("keys", static_cast<size_t>(sub) * key_stride * key_size, &keys));
  BVSS_TRY(alloc_select_state(idx, c));
  for (int q0 = 0; q0 < nq; q0 += static_cast<int>(sub)) {
    const int ns = static_cast<int>(q0 + sub <= nq ? sub : nq - q0);
    BVSS_TRY(scan_keys(idx, c, q0, ns, keys, key_stride));
    SelectState s2 = c->sel;
    s2.prefix += q0;
    s2.below += q0;
    s2.teff += q0;
    s2.eq += q0;
    s2.quota += q0;
    s2.digit += q0;
    BVSS_TRY(launch_select_init(s2, ns, c->teff, idx->stream));
    for (int r = 0; r < c->rounds; ++r) {
      BVSS_TRY(launch_select_hist(key_size, keys, key_stride, n, ns, s2, c->key_bits, r, c->local_hist, idx->stream));
      BVSS_TRY(launch_select_resolve(c->local_hist, s2, ns, c->key_bits, r, idx->stream));
    }
    BVSS_TRY(launch_select_bitmap(key_size, keys, key_stride, n, ns, s2, c->T, *mask + static_cast<int64_t>(q0) * words,
                                  words, idx->stream, key_limit_of(idx)));
    idx->stats.kernel_launches += 1 + 2 * c->rounds;
  }
  return BVSS_OK;
}

float ev_ms(bvss_index* idx, int a, int b) {
  float ms = 0.0f;
  if (cudaEventElapsedTime(&ms, idx->ev[a], idx->ev[b]) != cudaSuccess) return 0.0f;
  return ms;
}

int run_select_single(bvss_index* idx, bvss_search_ctx* c) {
  const int nq = static_cast<int>(c->nq);
  const int key_size = key_size_of(idx);
  for (int r = 0; r < c->rounds; ++r) {
    BVSS_TRY(launch_select_hist(key_size, c->keys, c->key_stride, idx->n, nq, c->sel, c->key_bits, r, c->local_hist,
                                idx->stream));
    BVSS_TRY(launch_select_resolve(c->local_hist, c->sel, nq, c->key_bits, r, idx->stream));
    idx->stats.kernel_launches += 2;
  }
  return BVSS_OK;
}

int make_ctx(bvss_index* idx, const float* queries, const std::vector<int64_t>& qoff_host, int k, int T,
             int64_t n_total, uint32_t flags, std::unique_ptr<bvss_search_ctx>& c, bool scan = true) {
  c.reset(new bvss_search_ctx());
  c->idx = idx;
  c->k = k;
  c->T = T;
  c->teff = T < n_total ? T : n_total;
  BVSS_TRY(prepare_queries(idx, c.get(), queries, qoff_host, (flags & BVSS_DEVICE_PTRS) != 0,
                           (flags & BVSS_VALIDATE_FINITE) != 0));
  if (scan) BVSS_TRY(scan_batch(idx, c.get()));
  return BVSS_OK;
}

int validate_search(bvss_index* idx, const float* q, const int64_t* qo, int64_t nq, int k, int T) {
  if (!idx) BVSS_FAIL(BVSS_EINVAL, "null index");
  if (idx->pending) BVSS_FAIL(BVSS_ESTATE, "streaming build not finished (bvss_index_finish)");
  if (!q || !qo) BVSS_FAIL(BVSS_EINVAL, "null query pointer");
  if (nq < 1) BVSS_FAIL(BVSS_EINVAL, "nq must be >= 1");
  if (k < 1) BVSS_FAIL(BVSS_EINVAL, "k must be >= 1");
  if (T < k) BVSS_FAIL(BVSS_EINVAL, "T (%d) < k (%d) (reading R16)", T, k);
  return BVSS_OK;
}

bool sampled_select_eligible(const bvss_index* idx);

int64_t batch_size(const bvss_index* idx, int64_t nq) {
  if (idx->query_batch) return idx->query_batch < nq ? idx->query_batch : nq;
  // sampled-threshold selection needs no key rows (its fallback runs in sub-batches): large batches
  if (sampled_select_eligible(idx)) return nq < 16384 ? nq : 16384;
  const int key_size = key_size_of(idx);
  const double per_q = static_cast<double>((idx->n + 7) & ~int64_t(7)) * key_size;
  int64_t b = static_cast<int64_t>((4.0 * (1ull << 30)) / per_q);
  if (b > 4096) b = 4096;
  if (b < 1) b = 1;
  return b < nq ? b : nq;
}

}  // namespace

// =================================================================== ABI ==
extern "C" {

const char* bvss_last_error(void) { return g_err; }

int bvss_device_count(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) return 0;
  int ok = 0;
  for (int i = 0; i < count; ++i) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, i) == cudaSuccess && p.major == 10) ++ok;
  }
  return ok;
}

}  // extern "C"

namespace {
// candidate-generation variants (gate.cu): stage-1 gate (A, M) and Alg 2
int validate_variants(const bvss_params* p) {
  if (p->filter > 1) BVSS_FAIL(BVSS_EINVAL, "filter must be 0 (sketch scan, Alg 6) or 1 (Haus^H over codes, Alg 2)");
  if (p->gate_A > 64 || p->gate_A > p->m) BVSS_FAIL(BVSS_EINVAL, "gate_A must be in [0, min(64, m)]");
  if (p->gate_A > 0 && p->gate_M > 255) BVSS_FAIL(BVSS_EINVAL, "gate_M must be <= 255 (u8 counters)");
  const bool binary = p->sketch == BVSS_SKETCH_BINARY || p->score == 2;
  if (p->gate_A > 0 && binary && p->gate_M > 1)
    BVSS_FAIL(BVSS_EINVAL, "a binary-sketch index holds no counts: the stage-1 gate needs gate_M <= 1 (S = (C > 0))");
  if (p->gate_A > 0 && p->score == 1) BVSS_FAIL(BVSS_EINVAL, "the stage-1 gate is not combined with the OVERLAP score");
  return BVSS_OK;
}

int validate_params(int64_t n, int32_t d, const bvss_params* p) {
  if (n < 1) BVSS_FAIL(BVSS_EINVAL, "n must be >= 1");
  if (d < 1 || d > 65535) BVSS_FAIL(BVSS_EINVAL, "d must be in [1, 65535]");
  if (p->m < 32 || p->m % 32 || p->m > 2048) BVSS_FAIL(BVSS_EINVAL, "m must be a multiple of 32 in [32, 2048]");
  if (p->L < 1 || p->L > p->m) BVSS_FAIL(BVSS_EINVAL, "L must be in [1, m]");
  if (p->s < 1 || static_cast<int>(p->s) > d || p->s > 32) BVSS_FAIL(BVSS_EINVAL, "s must be in [1, min(d, 32)]");
  if (p->sketch > 1) BVSS_FAIL(BVSS_EINVAL, "unknown sketch kind");
  if (p->refine_terms != 0 && p->refine_terms != 1 && p->refine_terms != 3 && p->refine_terms != 255)
    BVSS_FAIL(BVSS_EINVAL, "refine_terms must be 0 (default), 1, 3 or 255 (exact)");
  if (p->select_mode > 2) BVSS_FAIL(BVSS_EINVAL, "select_mode must be 0 (auto), 1 (full keys) or 2 (sampled)");
  if (p->metric > 2) BVSS_FAIL(BVSS_EINVAL, "metric must be 0 (Hausdorff), 1 (MeanMin) or 2 (Min)");
  if (p->score > 3) BVSS_FAIL(BVSS_EINVAL, "score must be 0 (Hamming / L2^2), 1 (OVERLAP), 2 (BINARIZED) or 3 (L1)");
  return validate_variants(p);
}

void free_index_resources(bvss_index* idx);

// Owns a partially built index: on any early return of the build its device buffers, stream and events are
// released (a failure after the stream was created leaked everything); an adopted vector buffer is
// left to the caller's handle, which still owns it until the build succeeds.
struct IndexGuard {
  bvss_index* p;
  float* adopted;
  ~IndexGuard() {
    if (!p) return;
    if (p->V == adopted) p->V = nullptr;
    free_index_resources(p);
    delete p;
  }
  bvss_index* operator->() const { return p; }
  bvss_index* release() {
    bvss_index* r = p;
    p = nullptr;
    return r;
  }
};

// The build (Algs 1, 3, 5).  adopt_V: a device buffer [nvec][d] the index takes over (streaming build) instead of
// copying `vectors`.
int build_impl(const float* vectors, const int64_t* set_offsets, int64_t n, int32_t d, const bvss_params* p,
               float* adopt_V, bvss_index** out) {
  if (!out) BVSS_FAIL(BVSS_EINVAL, "null out");
  *out = nullptr;
  if ((!vectors && !adopt_V) || !set_offsets || !p) BVSS_FAIL(BVSS_EINVAL, "null argument");
  if (n < 1) BVSS_FAIL(BVSS_EINVAL, "n must be >= 1");
  if (d < 1 || d > 65535) BVSS_FAIL(BVSS_EINVAL, "d must be in [1, 65535]");
  if (p->m < 32 || p->m % 32 || p->m > 2048) BVSS_FAIL(BVSS_EINVAL, "m must be a multiple of 32 in [32, 2048]");
  if (p->L < 1 || p->L > p->m) BVSS_FAIL(BVSS_EINVAL, "L must be in [1, m]");
  if (p->s < 1 || static_cast<int>(p->s) > d || p->s > 32) BVSS_FAIL(BVSS_EINVAL, "s must be in [1, min(d, 32)]");
  if (p->sketch > 1) BVSS_FAIL(BVSS_EINVAL, "unknown sketch kind");
  if (p->refine_terms != 0 && p->refine_terms != 1 && p->refine_terms != 3 && p->refine_terms != 255)
    BVSS_FAIL(BVSS_EINVAL, "refine_terms must be 0 (default), 1, 3 or 255 (exact)");
  if (p->select_mode > 2) BVSS_FAIL(BVSS_EINVAL, "select_mode must be 0 (auto), 1 (full keys) or 2 (sampled)");
  if (p->metric > 2) BVSS_FAIL(BVSS_EINVAL, "metric must be 0 (Hausdorff), 1 (MeanMin) or 2 (Min)");
  if (p->score > 3) BVSS_FAIL(BVSS_EINVAL, "score must be 0 (Hamming / L2^2), 1 (OVERLAP), 2 (BINARIZED) or 3 (L1)");
  BVSS_TRY(validate_variants(p));
  int num_sms = 0;
  BVSS_TRY(check_device(p->device, &num_sms));
  DeviceGuard g(p->device);
  const bool dev_ptrs = (p->flags & BVSS_DEVICE_PTRS) != 0;
  std::vector<int64_t> off_h(n + 1);
  if (dev_ptrs) {
    BVSS_CUDA(cudaMemcpy(off_h.data(), set_offsets, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));  // before any work
  } else {
    std::memcpy(off_h.data(), set_offsets, (n + 1) * sizeof(int64_t));
  }
  BVSS_TRY(check_offsets(off_h.data(), n, "database"));
  IndexGuard idx{new bvss_index(), adopt_V};
  idx->device = p->device;
  idx->num_sms = num_sms;
  idx->n = n;
  idx->nvec = off_h[n];
  idx->d = d;
  idx->dpad = (d + 63) / 64 * 64;
  idx->m = p->m;
  idx->s = p->s;
  idx->L = p->L;
  // BINARIZED (R25): Hamming on (C > 0) is Hamming on the OR-fold, so a count-sketch index scored
  // BINARIZED is built and scanned as a binary-sketch index
  idx->sketch = (p->sketch == BVSS_SKETCH_COUNT_U8 && p->score == 2) ? static_cast<uint32_t>(BVSS_SKETCH_BINARY) : p->sketch;
  idx->seed = p->seed;
  // 0 = default (1-term fp16 tensor-core pass + exact window), 1, 3, 255 = exact SIMT for every candidate
  idx->terms = p->refine_terms == 0 ? 1 : (p->refine_terms == 255 ? 0 : static_cast<int>(p->refine_terms));
  idx->query_batch = p->query_batch;
  idx->select_mode = p->select_mode;
  idx->metric = static_cast<int>(p->metric);
  idx->score = static_cast<int>(p->score);
  idx->gate_A = p->gate_A;
  idx->gate_M = p->gate_A > 0 ? p->gate_M : 0;
  idx->filter = p->filter;
  BVSS_CUDA(cudaStreamCreateWithFlags(&idx->own_stream, cudaStreamNonBlocking));
  idx->stream = idx->own_stream;
  for (auto& e : idx->ev) BVSS_CUDA(cudaEventCreate(&e));
  cudaStream_t st = idx->stream;
  const int64_t nvec = idx->nvec;
  const int R = p->m / 32;
  auto dalloc = [&](size_t bytes, void** ptr) -> int {
    BVSS_CUDA(cudaMalloc(ptr, bytes < 256 ? 256 : bytes));
    idx->owned_bytes += bytes;
    return BVSS_OK;
  };
  // projection
  if (p->projection) {
    idx->W.assign(p->projection, p->projection + static_cast<size_t>(p->m) * p->s);
    for (uint32_t j = 0; j < p->m; ++j)
      for (uint32_t t = 0; t < p->s; ++t) {
        const uint16_t v = idx->W[j * p->s + t];
        if (v >= d || (t > 0 && v <= idx->W[j * p->s + t - 1]))
          BVSS_FAIL(BVSS_EINVAL, "projection row %u must hold s sorted distinct dims < d", j);
      }
  } else {
    make_projection(p->seed, p->m, p->s, d, idx->W);
  }
  std::vector<uint16_t> Wt(static_cast<size_t>(p->m) * p->s);
  for (uint32_t j = 0; j < p->m; ++j)
    for (uint32_t t = 0; t < p->s; ++t) Wt[static_cast<size_t>(t) * p->m + j] = idx->W[static_cast<size_t>(j) * p->s + t];
  BVSS_TRY(dalloc(Wt.size() * 2, reinterpret_cast<void**>(&idx->Wt)));
  BVSS_CUDA(cudaMemcpyAsync(idx->Wt, Wt.data(), Wt.size() * 2, cudaMemcpyHostToDevice, idx->stream));
  BVSS_CUDA(cudaStreamSynchronize(idx->stream));
  // data
  if (adopt_V) {
    idx->V = adopt_V;
    idx->owned_bytes += static_cast<size_t>(nvec) * d * 4;
  } else {
    BVSS_TRY(dalloc(static_cast<size_t>(nvec) * d * 4, reinterpret_cast<void**>(&idx->V)));
  }
  BVSS_TRY(dalloc((n + 1) * 8, reinterpret_cast<void**>(&idx->off)));
  if (!adopt_V) BVSS_TRY(to_device(idx.p, idx->V, vectors, static_cast<size_t>(nvec) * d * 4, dev_ptrs));
  BVSS_CUDA(cudaMemcpyAsync(idx->off, off_h.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st));
  if (p->flags & BVSS_VALIDATE_FINITE) {
    int* bad;
    BVSS_TRY(idx->ws.get("bad", sizeof(int), reinterpret_cast<void**>(&bad)));
    BVSS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    BVSS_TRY(launch_finite_check(idx->V, nvec * d, bad, num_sms, st));
    int hbad = 0;
    BVSS_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    BVSS_CUDA(cudaStreamSynchronize(st));
    if (hbad) BVSS_FAIL(BVSS_ENONFINITE, "database vectors contain NaN or Inf");
  }
  // refine operands: every set starts on an 8-aligned padded row (refine.cu)
  std::vector<int64_t> pb(n + 1);
  pb[0] = 0;
  for (int64_t i = 0; i < n; ++i) pb[i + 1] = pb[i] + ((off_h[i + 1] - off_h[i] + 7) & ~int64_t(7));
  idx->prows = pb[n];
  idx->off_h = off_h;
  for (int64_t i = 0; i < n; ++i)
    idx->max_rows = static_cast<int>(std::max<int64_t>(idx->max_rows, std::min<int64_t>(off_h[i + 1] - off_h[i], 1 << 30)));
  BVSS_TRY(dalloc((n + 1) * 8, reinterpret_cast<void**>(&idx->pbase)));
  BVSS_CUDA(cudaMemcpyAsync(idx->pbase, pb.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st));
  BVSS_TRY(dalloc(static_cast<size_t>(idx->prows) * idx->dpad * 2, reinterpret_cast<void**>(&idx->hi)));
  if (idx->terms == 3)  // the lo piece of the fp16 split is read only by the 3-term Gram
    BVSS_TRY(dalloc(static_cast<size_t>(idx->prows) * idx->dpad * 2, reinterpret_cast<void**>(&idx->lo)));
  BVSS_TRY(dalloc(static_cast<size_t>(idx->prows) * 4, reinterpret_cast<void**>(&idx->vscale)));
  BVSS_CUDA(cudaMemsetAsync(idx->vscale, 0, static_cast<size_t>(idx->prows) * 4, st));
  BVSS_CUDA(cudaMemsetAsync(idx->hi, 0, static_cast<size_t>(idx->prows) * idx->dpad * 2, st));
  if (idx->lo) BVSS_CUDA(cudaMemsetAsync(idx->lo, 0, static_cast<size_t>(idx->prows) * idx->dpad * 2, st));
  int64_t* dst_row;
  BVSS_TRY(idx->ws.get("dst_row", static_cast<size_t>(nvec) * 8, reinterpret_cast<void**>(&dst_row)));
  pad_rows_kernel<<<num_sms * 8, 256, 0, st>>>(idx->off, idx->pbase, n, dst_row);
  BVSS_TRY(post_launch("pad_rows_kernel", st));
  BVSS_TRY(dalloc(static_cast<size_t>(nvec) * 4, reinterpret_cast<void**>(&idx->vnorm)));
  uint32_t* codes = nullptr;
  const bool keep = (p->flags & BVSS_KEEP_CODES) != 0 || p->filter == 1;  // Alg 2 scans the per-vector codes
  if (keep) {
    BVSS_TRY(dalloc(static_cast<size_t>(nvec) * R * 4, reinterpret_cast<void**>(&idx->codes)));
    codes = idx->codes;
  } else {
    BVSS_TRY(idx->ws.get("codes", static_cast<size_t>(nvec) * R * 4, reinterpret_cast<void**>(&codes)));
  }
  BVSS_TRY(launch_encode(idx->V, nvec, d, idx->Wt, p->m, p->s, p->L, codes, idx->vnorm, idx->hi, idx->lo, idx->vscale,
                         idx->dpad, idx->prows, dst_row, refine_kcs(idx->dpad), num_sms, st));
  const int cps = chunks_per_set(idx.p);
  BVSS_TRY(dalloc(static_cast<size_t>(n) * cps * 16, &idx->sk));
  BVSS_TRY(dalloc(static_cast<size_t>(n) * 4, reinterpret_cast<void**>(&idx->mass)));
  BVSS_TRY(launch_sketch(codes, p->m, idx->off, n, idx->sketch, idx->sk, idx->mass, n, 1, num_sms, st));
  if (idx->score == 1) BVSS_CUDA(cudaMemsetAsync(idx->mass, 0, static_cast<size_t>(n) * 4, st));  // OVERLAP (R24)
  if (gated(idx.p)) {  // stage-1 gate (gate.cu): one bit plane per position, bit i = (C_i[p] >= M)
    idx->gW = (n + 31) / 32;
    BVSS_TRY(dalloc(static_cast<size_t>(p->m) * idx->gW * 4, reinterpret_cast<void**>(&idx->planes)));
    BVSS_TRY(launch_gate_planes(idx->sk, n, static_cast<int>(p->m), static_cast<int>(idx->sketch),
                                static_cast<int>(idx->gate_M), idx->planes, idx->gW, num_sms, st));
  }
  if (use_tc_scan(idx.p)) {
    // strided database sample for the sampled-threshold select
    idx->ns = n < 16384 ? n : 16384;
    BVSS_TRY(dalloc(static_cast<size_t>(idx->ns) * cps * 16, &idx->smp_sk));
    BVSS_TRY(dalloc(static_cast<size_t>(idx->ns) * 4, reinterpret_cast<void**>(&idx->smp_mass)));
    BVSS_TRY(launch_gather_sample(idx->sk, idx->mass, n, cps, idx->ns, idx->smp_sk, idx->smp_mass, num_sms, st));
    if (idx->sketch == BVSS_SKETCH_BINARY) {  // FP4 tensor-core operands (m/2 bytes per set)
      BVSS_TRY(dalloc(static_cast<size_t>(n) * p->m / 2, &idx->skx));
      BVSS_TRY(dalloc(static_cast<size_t>(idx->ns) * p->m / 2, &idx->smp_skx));
      BVSS_TRY(launch_expand_db_fp4(idx->sk, n, n, p->m, idx->skx, num_sms, st));
      BVSS_TRY(launch_expand_db_fp4(idx->smp_sk, idx->ns, idx->ns, p->m, idx->smp_skx, num_sms, st));
    }
  }
  unsigned int* vmax;
  BVSS_TRY(idx->ws.get("vmax", sizeof(unsigned int), reinterpret_cast<void**>(&vmax)));
  BVSS_CUDA(cudaMemsetAsync(vmax, 0, sizeof(unsigned int), st));
  max_float_kernel<<<num_sms * 2, 256, 0, st>>>(idx->vnorm, nvec, vmax);
  BVSS_TRY(post_launch("max_float_kernel", st));
  unsigned int hv = 0;
  BVSS_CUDA(cudaMemcpyAsync(&hv, vmax, sizeof(hv), cudaMemcpyDeviceToHost, st));
  BVSS_CUDA(cudaStreamSynchronize(st));
  std::memcpy(&idx->vmax2, &hv, 4);
  idx->ws.release();  // build scratch (codes unless kept, padded-row map)
  *out = idx.release();
  return BVSS_OK;
}
}  // namespace

extern "C" {

int bvss_build_index(const float* vectors, const int64_t* set_offsets, int64_t n, int32_t d, const bvss_params* p,
                     bvss_index** out) {
  return build_impl(vectors, set_offsets, n, d, p, nullptr, out);
}

int bvss_index_begin(int64_t n_total, int64_t nvec_total, int32_t d, const bvss_params* p, bvss_index** out) {
  if (!out || !p) BVSS_FAIL(BVSS_EINVAL, "null argument");
  *out = nullptr;
  BVSS_TRY(validate_params(n_total, d, p));
  if (nvec_total < n_total) BVSS_FAIL(BVSS_EINVAL, "nvec_total < n_total (every set has >= 1 vector)");
  int num_sms = 0;
  BVSS_TRY(check_device(p->device, &num_sms));
  DeviceGuard g(p->device);
  IndexGuard idx{new bvss_index(), nullptr};  // a failed allocation below releases the stream too
  idx->pending = true;
  idx->device = p->device;
  idx->num_sms = num_sms;
  idx->n_total = n_total;
  idx->nvec_total = nvec_total;
  idx->d = d;
  idx->pend_p = *p;
  if (p->projection) {
    idx->pend_proj.assign(p->projection, p->projection + static_cast<size_t>(p->m) * p->s);
    idx->pend_p.projection = idx->pend_proj.data();
  }
  idx->pend_off.assign(1, 0);
  idx->pend_off.reserve(n_total + 1);
  BVSS_CUDA(cudaStreamCreateWithFlags(&idx->own_stream, cudaStreamNonBlocking));
  idx->stream = idx->own_stream;
  BVSS_CUDA(cudaMalloc(reinterpret_cast<void**>(&idx->pend_V), static_cast<size_t>(nvec_total) * d * 4));
  *out = idx.release();
  return BVSS_OK;
}

int bvss_index_append(bvss_index* idx, const float* vectors, const int64_t* local_offsets, int64_t n_chunk) {
  if (!idx || !vectors || !local_offsets) BVSS_FAIL(BVSS_EINVAL, "null argument");
  if (!idx->pending) BVSS_FAIL(BVSS_ESTATE, "index is not in a streaming build");
  if (n_chunk < 1) BVSS_FAIL(BVSS_EINVAL, "n_chunk must be >= 1");
  DeviceGuard g(idx->device);
  const bool dev = (idx->pend_p.flags & BVSS_DEVICE_PTRS) != 0;
  std::vector<int64_t> lo(n_chunk + 1);
  if (dev) {
    BVSS_CUDA(cudaMemcpy(lo.data(), local_offsets, (n_chunk + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
  } else {
    std::memcpy(lo.data(), local_offsets, (n_chunk + 1) * sizeof(int64_t));
  }
  BVSS_TRY(check_offsets(lo.data(), n_chunk, "chunk"));
  if (idx->n_appended + n_chunk > idx->n_total || idx->nvec_appended + lo[n_chunk] > idx->nvec_total)
    BVSS_FAIL(BVSS_EINVAL, "chunk exceeds the sizes declared at bvss_index_begin");
  BVSS_CUDA(cudaMemcpyAsync(idx->pend_V + idx->nvec_appended * idx->d, vectors,
                            static_cast<size_t>(lo[n_chunk]) * idx->d * 4,
                            dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, idx->stream));
  BVSS_CUDA(cudaStreamSynchronize(idx->stream));  // the caller may reuse its chunk buffers on return
  for (int64_t i = 1; i <= n_chunk; ++i) idx->pend_off.push_back(idx->nvec_appended + lo[i]);
  idx->n_appended += n_chunk;
  idx->nvec_appended += lo[n_chunk];
  return BVSS_OK;
}

int bvss_index_finish(bvss_index* idx) {
  if (!idx) BVSS_FAIL(BVSS_EINVAL, "null index");
  if (!idx->pending) BVSS_FAIL(BVSS_ESTATE, "index is not in a streaming build");
  if (idx->n_appended != idx->n_total || idx->nvec_appended != idx->nvec_total)
    BVSS_FAIL(BVSS_EINVAL, "appended %lld sets / %lld vectors, declared %lld / %lld",
              static_cast<long long>(idx->n_appended), static_cast<long long>(idx->nvec_appended),
              static_cast<long long>(idx->n_total), static_cast<long long>(idx->nvec_total));
  DeviceGuard g(idx->device);
  bvss_params p = idx->pend_p;
  p.flags &= ~BVSS_DEVICE_PTRS;  // offsets are host-side now; vectors are adopted
  bvss_index* built = nullptr;
  BVSS_TRY(build_impl(nullptr, idx->pend_off.data(), idx->n_total, idx->d, &p, idx->pend_V, &built));
  idx->pend_V = nullptr;  // owned by `built` now
  // move the built state into the caller's handle
  cudaStream_t old_stream = idx->own_stream;
  *idx = std::move(*built);
  built->own_stream = nullptr;
  built->V = nullptr;
  built->off = nullptr;
  built->Wt = nullptr;
  built->hi = built->lo = nullptr;
  built->vscale = built->vnorm = nullptr;
  built->pbase = nullptr;
  built->codes = nullptr;
  built->sk = built->smp_sk = built->skx = built->smp_skx = nullptr;
  built->mass = built->smp_mass = nullptr;
  built->hd = built->va = nullptr;
  built->planes = nullptr;
  built->dtile_s0 = built->dtile_s1 = built->dhuge = nullptr;
  for (auto& e : built->ev) e = nullptr;
  delete built;
  if (old_stream) cudaStreamDestroy(old_stream);
  return BVSS_OK;
}

void bvss_free_index(bvss_index* idx) {
  if (!idx) return;
  free_index_resources(idx);
  delete idx;
}

}  // extern "C"

namespace {
void free_index_resources(bvss_index* idx) {
  DeviceGuard g(idx->device);
  if (idx->stream) cudaStreamSynchronize(idx->stream);
  void* ptrs[] = {idx->Wt,    idx->V,     idx->off,   idx->hi,   idx->lo,     idx->vscale, idx->pbase,
                  idx->vnorm, idx->codes, idx->sk,    idx->mass, idx->smp_sk, idx->smp_mass,
                  idx->skx,   idx->smp_skx, idx->hd, idx->va, idx->dtile_s0, idx->dtile_s1, idx->dhuge,
                  idx->planes};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (idx->pend_V) cudaFree(idx->pend_V);
  idx->ws.release();
  for (auto& e : idx->ev)
    if (e) cudaEventDestroy(e);
  if (idx->own_stream) cudaStreamDestroy(idx->own_stream);
  idx->own_stream = idx->stream = nullptr;
}
}  // namespace

extern "C" {

int bvss_set_stream(bvss_index* idx, void* stream) {
  if (!idx) BVSS_FAIL(BVSS_EINVAL, "null index");
  idx->stream = stream ? static_cast<cudaStream_t>(stream) : idx->own_stream;
  return BVSS_OK;
}

int bvss_get_info(const bvss_index* idx, bvss_info* out) {
  if (!idx || !out) BVSS_FAIL(BVSS_EINVAL, "null argument");
  out->n = idx->n;
  out->nvec = idx->nvec;
  out->d = idx->d;
  out->dpad = idx->dpad;
  out->m = idx->m;
  out->s = idx->s;
  out->L = idx->L;
  out->sketch = idx->sketch;
  out->device = idx->device;
  out->device_bytes = idx->owned_bytes;
  out->workspace_bytes = idx->ws.total;
  return BVSS_OK;
}

int bvss_get_stats(const bvss_index* idx, bvss_stats* out) {
  if (!idx || !out) BVSS_FAIL(BVSS_EINVAL, "null argument");
  *out = idx->stats;
  return BVSS_OK;
}

double bvss_refine_error_bound(const bvss_index* idx, double qnorm_max) {
  if (!idx) return -1.0;
  float c1, c2;
  error_consts(idx, &c1, &c2);
  const double mv = std::sqrt(static_cast<double>(idx->vmax2));
  return c1 * qnorm_max * mv + c2 * (qnorm_max * qnorm_max + idx->vmax2);
}

int bvss_export_projection(const bvss_index* idx, uint16_t* out) {
  if (!idx || !out) BVSS_FAIL(BVSS_EINVAL, "null argument");
  std::memcpy(out, idx->W.data(), idx->W.size() * 2);
  return BVSS_OK;
}

int bvss_export_codes(const bvss_index* idx, int64_t first, int64_t count, uint32_t* out) {
  if (!idx || !out) BVSS_FAIL(BVSS_EINVAL, "null argument");
  if (!idx->codes) BVSS_FAIL(BVSS_ESTATE, "index was built without BVSS_KEEP_CODES");
  if (first < 0 || count < 0 || first + count > idx->nvec) BVSS_FAIL(BVSS_EINVAL, "vector range out of bounds");
  DeviceGuard g(idx->device);
  const size_t R = idx->m / 32;
  BVSS_CUDA(cudaMemcpyAsync(out, idx->codes + first * R, count * R * 4, cudaMemcpyDeviceToHost, idx->stream));
  BVSS_CUDA(cudaStreamSynchronize(idx->stream));
  return BVSS_OK;
}

int bvss_export_sketches(const bvss_index* idx_c, int64_t first, int64_t count, void* out) {
  bvss_index* idx = const_cast<bvss_index*>(idx_c);
  if (!idx || !out) BVSS_FAIL(BVSS_EINVAL, "null argument");
  if (first < 0 || count < 0 || first + count > idx->n) BVSS_FAIL(BVSS_EINVAL, "set range out of bounds");
  DeviceGuard g(idx->device);
  const int words = idx->sketch == BVSS_SKETCH_BINARY ? static_cast<int>(idx->m / 32) : static_cast<int>(idx->m / 4);
  uint32_t* tmp;
  BVSS_TRY(idx->ws.get("export", static_cast<size_t>(count) * words * 4, reinterpret_cast<void**>(&tmp)));
  BVSS_TRY(launch_unchunk(idx->sk, idx->n, first, count, words, tmp, idx->stream));
  BVSS_CUDA(cudaMemcpyAsync(out, tmp, static_cast<size_t>(count) * words * 4, cudaMemcpyDeviceToHost, idx->stream));
  BVSS_CUDA(cudaStreamSynchronize(idx->stream));
  return BVSS_OK;
}

int bvss_query_sketch(bvss_index* idx, const float* queries, const int64_t* query_offsets, int64_t nq, void* out_sketch,
                      uint32_t* out_codes, uint32_t flags) {
  if (!idx || !queries || !query_offsets || !out_sketch) BVSS_FAIL(BVSS_EINVAL, "null argument");
  if (nq < 1) BVSS_FAIL(BVSS_EINVAL, "nq must be >= 1");
  DeviceGuard g(idx->device);
  const bool dev = (flags & BVSS_DEVICE_PTRS) != 0;
  std::vector<int64_t> qo;
  BVSS_TRY(host_offsets(idx, query_offsets, nq, dev, qo));
  std::unique_ptr<bvss_search_ctx> c(new bvss_search_ctx());
  c->idx = idx;
  BVSS_TRY(prepare_queries(idx, c.get(), queries, qo, dev, (flags & BVSS_VALIDATE_FINITE) != 0));
  const int cps = chunks_per_set(idx);
  const size_t row_bytes = idx->sketch == BVSS_SKETCH_BINARY ? idx->m / 8 : idx->m;
  BVSS_CUDA(cudaMemcpy2DAsync(out_sketch, row_bytes, c->qsk, static_cast<size_t>(cps) * 16, row_bytes, nq,
                              dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, idx->stream));
  if (out_codes)
    BVSS_TRY(from_device(idx, out_codes, c->qcodes, static_cast<size_t>(c->nqvec) * (idx->m / 32) * 4, dev));
  BVSS_CUDA(cudaStreamSynchronize(idx->stream));
  return BVSS_OK;
}

int bvss_filter(bvss_index* idx, const float* queries, const int64_t* query_offsets, int64_t nq, int32_t T,
                int32_t* out_cand, int32_t* out_score, uint32_t flags) {
  BVSS_TRY(validate_search(idx, queries, query_offsets, nq, 1, T));
  if (!out_cand) BVSS_FAIL(BVSS_EINVAL, "null out_cand");
  DeviceGuard g(idx->device);
  const bool dev = (flags & BVSS_DEVICE_PTRS) != 0;
  std::vector<int64_t> qo;
  BVSS_TRY(host_offsets(idx, query_offsets, nq, dev, qo));
  std::unique_ptr<bvss_search_ctx> c;
  BVSS_TRY(make_ctx(idx, queries, qo, 1, T, idx->n, flags, c));
  BVSS_TRY(run_select_single(idx, c.get()));
  const int key_size = key_size_of(idx);
  int32_t *cand, *score;
  BVSS_TRY(c->alloc(static_cast<size_t>(nq) * T * 4, reinterpret_cast<void**>(&cand)));
  BVSS_TRY(c->alloc(static_cast<size_t>(nq) * T * 4, reinterpret_cast<void**>(&score)));
  BVSS_TRY(launch_select_emit(key_size, c->keys, c->key_stride, idx->n, static_cast<int>(nq), c->sel, T, 0, cand, score,
                              nullptr, idx->stream, key_limit_of(idx)));
  BVSS_TRY(from_device(idx, out_cand, cand, static_cast<size_t>(nq) * T * 4, dev));
  if (out_score) BVSS_TRY(from_device(idx, out_score, score, static_cast<size_t>(nq) * T * 4, dev));
  BVSS_CUDA(cudaStreamSynchronize(idx->stream));
  return BVSS_OK;
}

// K8 brute force ("precise calculations according to Definition 4"): the exact top-k over the first
// set_limit sets, as chunks of the refine path (tensor-core Hausdorff + exact fix-up window, which is exact)
// merged by K7.
int bvss_bruteforce(bvss_index* idx, const float* queries, const int64_t* query_offsets, int64_t nq,
                    int64_t set_limit, int32_t k, int64_t* out_ids, float* out_dist, uint32_t flags) {
  BVSS_TRY(validate_search(idx, queries, query_offsets, nq, k, k));
  if (!out_ids || !out_dist) BVSS_FAIL(BVSS_EINVAL, "null output");
  DeviceGuard g(idx->device);
  const bool dev = (flags & BVSS_DEVICE_PTRS) != 0;
  std::vector<int64_t> qo;
  BVSS_TRY(host_offsets(idx, query_offsets, nq, dev, qo));
  const int64_t lim = (set_limit <= 0 || set_limit > idx->n) ? idx->n : set_limit;
  if (dense_wanted(idx, idx->n)) {  // K8 on the dense kernel (dense.cu): one pass over the first lim sets
    std::unique_ptr<bvss_search_ctx> c(new bvss_search_ctx());
    c->idx = idx;
    c->k = k;
    c->T = static_cast<int>(lim < (1ll << 30) ? lim : (1ll << 30));
    idx->stats = bvss_stats{};
    BVSS_TRY(prepare_queries(idx, c.get(), queries, qo, dev, (flags & BVSS_VALIDATE_FINITE) != 0));
    if (dense_supported(idx, c.get())) {
      BVSS_TRY(ensure_dense(idx));
      int nt = idx->dntiles;
      uint32_t* mask = nullptr;
      if (lim < idx->n) {  // tiles up to the one holding set lim - 1, and a shared bitmap of the sets < lim
        nt = static_cast<int>(std::upper_bound(idx->dtile_s0_h.begin(), idx->dtile_s0_h.end(),
                                               static_cast<int32_t>(lim - 1)) - idx->dtile_s0_h.begin());
        const int64_t words = (idx->n + 31) / 32;
        std::vector<uint32_t> row(words, 0u);
        for (int64_t i = 0; i < lim; ++i) row[i >> 5] |= 1u << (i & 31);
        BVSS_TRY(c->alloc(words * 4, reinterpret_cast<void**>(&mask)));
        BVSS_CUDA(cudaMemcpyAsync(mask, row.data(), words * 4, cudaMemcpyHostToDevice, idx->stream));
        BVSS_CUDA(cudaStreamSynchronize(idx->stream));
      }
      int64_t* oi;
      float* od;
      BVSS_TRY(c->alloc(static_cast<size_t>(nq) * k * 8, reinterpret_cast<void**>(&oi)));
      BVSS_TRY(c->alloc(static_cast<size_t>(nq) * k * 4, reinterpret_cast<void**>(&od)));
      bool done = false;
      BVSS_TRY(dense_refine_topk(idx, c.get(), mask, 0, nt, oi, od, &done));
      if (done) {
        BVSS_TRY(from_device(idx, out_ids, oi, static_cast<size_t>(nq) * k * 8, dev));
        BVSS_TRY(from_device(idx, out_dist, od, static_cast<size_t>(nq) * k * 4, dev));
        BVSS_CUDA(cudaStreamSynchronize(idx->stream));
        idx->stats.ms_refine = ev_ms(idx, 4, 5);
        idx->stats.ms_topk = ev_ms(idx, 5, 6);
        return BVSS_OK;
      }
    }
  }
  std::unique_ptr<bvss_search_ctx> c(new bvss_search_ctx());
  c->idx = idx;
  c->k = k;
  const int chunk = static_cast<int>(lim < 8192 ? (lim < k ? k : lim) : 8192);
  c->T = chunk;
  BVSS_TRY(prepare_queries(idx, c.get(), queries, qo, dev, (flags & BVSS_VALIDATE_FINITE) != 0));
  BVSS_TRY(c->alloc(static_cast<size_t>(nq) * chunk * 4, reinterpret_cast<void**>(&c->cand)));
  BVSS_TRY(c->alloc(nq * 4, reinterpret_cast<void**>(&c->count)));
  int64_t *ids[3];
  float* dd[3];
  for (int b = 0; b < 3; ++b) {  // [0] running, [1] chunk (contiguous after [0] for the 2-way merge), [2] merged
    BVSS_TRY(c->alloc(static_cast<size_t>(nq) * k * 8 * (b == 0 ? 2 : 1), reinterpret_cast<void**>(&ids[b])));
    BVSS_TRY(c->alloc(static_cast<size_t>(nq) * k * 4 * (b == 0 ? 2 : 1), reinterpret_cast<void**>(&dd[b])));
  }
  int64_t* run_i = ids[0];
  float* run_d = dd[0];
  int64_t* chk_i = ids[0] + static_cast<int64_t>(nq) * k;
  float* chk_d = dd[0] + static_cast<int64_t>(nq) * k;
  for (int64_t c0 = 0; c0 < lim; c0 += chunk) {
    const int cnt = static_cast<int>(c0 + chunk <= lim ? chunk : lim - c0);
    fill_range_kernel<<<idx->num_sms * 4, 256, 0, idx->stream>>>(c->cand, c->count, static_cast<int>(nq), chunk, c0,
                                                                  cnt);
    BVSS_TRY(post_launch("fill_range_kernel", idx->stream));
    BVSS_TRY(refine_topk(idx, c.get(), c0 == 0 ? run_i : chk_i, c0 == 0 ? run_d : chk_d));
    if (c0 > 0) {
      BVSS_TRY(launch_merge_topk(run_i, run_d, 2, nq, k, ids[1], dd[1], idx->stream));
      BVSS_CUDA(cudaMemcpyAsync(run_i, ids[1], static_cast<size_t>(nq) * k * 8, cudaMemcpyDeviceToDevice, idx->stream));
      BVSS_CUDA(cudaMemcpyAsync(run_d, dd[1], static_cast<size_t>(nq) * k * 4, cudaMemcpyDeviceToDevice, idx->stream));
    }
  }
  BVSS_TRY(from_device(idx, out_ids, run_i, static_cast<size_t>(nq) * k * 8, dev));
  BVSS_TRY(from_device(idx, out_dist, run_d, static_cast<size_t>(nq) * k * 4, dev));
  BVSS_CUDA(cudaStreamSynchronize(idx->stream));
  return BVSS_OK;
}

int bvss_refine(bvss_index* idx, const float* queries, const int64_t* query_offsets, int64_t nq, const int32_t* cand,
                int32_t T, int32_t k, int64_t* out_ids, float* out_dist, float* out_approx, uint32_t flags) {
  BVSS_TRY(validate_search(idx, queries, query_offsets, nq, k, T < k ? k : T));
  if (!cand || !out_ids || !out_dist) BVSS_FAIL(BVSS_EINVAL, "null argument");
  DeviceGuard g(idx->device);
  const bool dev = (flags & BVSS_DEVICE_PTRS) != 0;
  std::vector<int64_t> qo;
  BVSS_TRY(host_offsets(idx, query_offsets, nq, dev, qo));
  std::unique_ptr<bvss_search_ctx> c(new bvss_search_ctx());
  c->idx = idx;
  c->k = k;
  c->T = T;
  BVSS_TRY(prepare_queries(idx, c.get(), queries, qo, dev, (flags & BVSS_VALIDATE_FINITE) != 0));
  BVSS_TRY(c->alloc(static_cast<size_t>(nq) * T * 4, reinterpret_cast<void**>(&c->cand)));
  BVSS_TRY(c->alloc(nq * 4, reinterpret_cast<void**>(&c->count)));
  BVSS_TRY(to_device(idx, c->cand, cand, static_cast<size_t>(nq) * T * 4, dev));
  count_valid_kernel<<<static_cast<int>(nq), 256, 0, idx->stream>>>(c->cand, T, static_cast<int>(nq), c->count);
  BVSS_TRY(post_launch("count_valid_kernel", idx->stream));
  int64_t* oid;
  float* odist;
  BVSS_TRY(c->alloc(static_cast<size_t>(nq) * k * 8, reinterpret_cast<void**>(&oid)));
  BVSS_TRY(c->alloc(static_cast<size_t>(nq) * k * 4, reinterpret_cast<void**>(&odist)));
  int exact_all = 0;
  float c1, c2;
  error_consts(idx, &c1, &c2);
  if (idx->terms != 0) {  // tensor path (query sets > 128 rows: per query on the exact path, refine.cu)
    BVSS_TRY(c->alloc(static_cast<size_t>(nq) * T * 4, reinterpret_cast<void**>(&c->approx)));
    BVSS_CUDA(cudaMemsetAsync(c->approx, 0xFF, static_cast<size_t>(nq) * T * 4, idx->stream));  // NaN where unused
    if (idx->metric == 1)
      BVSS_TRY(c->alloc(static_cast<size_t>(nq) * T * 4, reinterpret_cast<void**>(&c->approx_err)));
    int* counter;
    BVSS_TRY(idx->ws.get("work_counter", sizeof(int), reinterpret_cast<void**>(&counter)));
    BVSS_TRY(launch_refine_tc(idx->hi, idx->lo, idx->vscale, idx->prows, idx->pbase, idx->vnorm, idx->off, idx->dpad, c->qhi,
                              c->qlo, c->qscale, c->qrows,
                              c->qrow, c->qnorm, c->qoff, c->max_mq, c->cand, c->count, T, static_cast<int>(nq), 0,
                              c->approx, idx->terms, counter, nullptr, idx->num_sms,
                              0 /* caller lists: any order */, nullptr, idx->metric, c->approx_err, c1, c2,
                              idx->vmax2, idx->stream));
  } else {
    exact_all = 1;
  }
  void* scratch;
  BVSS_TRY(idx->ws.get("topk_scratch", static_cast<size_t>(nq) * T * 8, &scratch));
  BVSS_TRY(launch_topk_fixup(c->approx, c->cand, c->count, T, k, idx->V, idx->off, 0, idx->d, c->qv, c->qoff, c->qnorm,
                             idx->vmax2, c1, c2, exact_all, oid, odist, static_cast<int>(nq), nullptr, scratch,
                             idx->metric, c->approx_err, idx->max_rows, c->max_mq, idx->stream));
  BVSS_TRY(from_device(idx, out_ids, oid, static_cast<size_t>(nq) * k * 8, dev));
  BVSS_TRY(from_device(idx, out_dist, odist, static_cast<size_t>(nq) * k * 4, dev));
  if (out_approx && c->approx) BVSS_TRY(from_device(idx, out_approx, c->approx, static_cast<size_t>(nq) * T * 4, dev));
  BVSS_CUDA(cudaStreamSynchronize(idx->stream));
  return BVSS_OK;
}

int bvss_search(bvss_index* idx, const float* queries, const int64_t* query_offsets, int64_t nq, int32_t k, int32_t T,
                int64_t* out_ids, float* out_dist, uint32_t flags) {
  const auto t_entry = std::chrono::steady_clock::now();
  BVSS_TRY(validate_search(idx, queries, query_offsets, nq, k, T));
  if (!out_ids || !out_dist) BVSS_FAIL(BVSS_EINVAL, "null output");
  DeviceGuard g(idx->device);
  const bool dev = (flags & BVSS_DEVICE_PTRS) != 0;
  std::vector<int64_t> qo;
  BVSS_TRY(host_offsets(idx, query_offsets, nq, dev, qo));
  idx->stats = bvss_stats{};
  const int64_t B = batch_size(idx, nq);
  idx->stats.query_batch = static_cast<int32_t>(B);
  int64_t* oid;
  float* odist;
  BVSS_TRY(idx->ws.get("out_ids", static_cast<size_t>(B) * k * 8, reinterpret_cast<void**>(&oid)));
  BVSS_TRY(idx->ws.get("out_dist", static_cast<size_t>(B) * k * 4, reinterpret_cast<void**>(&odist)));
  int64_t* fix;
  unsigned long long* rows;
  BVSS_TRY(idx->ws.get("rows_counter", sizeof(unsigned long long), reinterpret_cast<void**>(&rows)));
  BVSS_CUDA(cudaMemsetAsync(rows, 0, sizeof(unsigned long long), idx->stream));
  float ms[6] = {0, 0, 0, 0, 0, 0};
  float tot = 0.0f;
  uint64_t fixups = 0;
  static const bool trace = getenv("BVSS_TRACE") != nullptr;  // developer switch: host-side phase timing
  auto now_us = [] { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double t_start = now_us();
  if (trace)
    fprintf(stderr, "[bvss] search entry -> batches %.0f us\n",
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_entry).count());
  for (int64_t b0 = 0; b0 < nq; b0 += B) {
    const int64_t nb = (b0 + B <= nq) ? B : nq - b0;
    const double t_b = now_us();
    std::vector<int64_t> sub(nb + 1);
    for (int64_t i = 0; i <= nb; ++i) sub[i] = qo[b0 + i] - qo[b0];
    std::unique_ptr<bvss_search_ctx> c;
    const bool sampled = sampled_select_eligible(idx);
    const int64_t teff = T < idx->n ? T : idx->n;
    const bool try_dense = dense_wanted(idx, teff);
    BVSS_TRY(make_ctx(idx, queries + qo[b0] * idx->d, sub, k, T, idx->n, flags, c, !sampled && !try_dense));
    bool done = false;
    double t_sel = 0.0;
    if (try_dense && dense_supported(idx, c.get())) {
      // candidate-major refine (dense.cu): the candidate set as a bitmap (none when T >= n), one dense pass
      uint32_t* mask = nullptr;
      int64_t mstride = 0;
      if (teff < idx->n) BVSS_TRY(dense_mask(idx, c.get(), &mask, &mstride));
      cudaEventRecord(idx->ev[3], idx->stream);
      t_sel = now_us();
      BVSS_TRY(dense_refine_topk(idx, c.get(), mask, mstride, -1, oid, odist, &done));
      if (!done && !sampled) BVSS_TRY(scan_batch(idx, c.get()));  // overflow: the query-major path below
    } else if (try_dense && !sampled) {
      BVSS_TRY(scan_batch(idx, c.get()));
    }
    if (!done) {
      bool ok = false;
      if (sampled) BVSS_TRY(select_sampled(idx, c.get(), &ok));
      if (!ok) {
        if (sampled) {
          BVSS_TRY(fallback_full(idx, c.get()));
        } else {
          BVSS_TRY(run_select_single(idx, c.get()));
          BVSS_TRY(emit_candidates(idx, c.get()));
        }
      }
      t_sel = now_us();
      BVSS_TRY(refine_topk(idx, c.get(), oid, odist));
    }
    const double t_ref = now_us();
    BVSS_TRY(from_device(idx, out_ids + b0 * k, oid, static_cast<size_t>(nb) * k * 8, dev));
    BVSS_TRY(from_device(idx, out_dist + b0 * k, odist, static_cast<size_t>(nb) * k * 4, dev));
    BVSS_CUDA(cudaEventRecord(idx->ev[7], idx->stream));
    BVSS_CUDA(cudaStreamSynchronize(idx->stream));
    for (int i = 0; i < 6; ++i) ms[i] += ev_ms(idx, i, i + 1);
    tot += ev_ms(idx, 0, 7);
    BVSS_TRY(idx->ws.get("fixup_counter", sizeof(int64_t), reinterpret_cast<void**>(&fix)));
    int64_t hf = 0;
    BVSS_CUDA(cudaMemcpyAsync(&hf, fix, sizeof(hf), cudaMemcpyDeviceToHost, idx->stream));
    BVSS_CUDA(cudaStreamSynchronize(idx->stream));
    fixups += static_cast<uint64_t>(hf);
    if (trace)
      fprintf(stderr, "[bvss] batch %lld: host issue->select %.0f us, refine issue %.0f us, wait %.0f us; gpu %.0f us\n",
              static_cast<long long>(b0), t_sel - t_b, t_ref - t_sel, now_us() - t_ref, 1000.0 * ev_ms(idx, 0, 7));
  }
  if (trace) fprintf(stderr, "[bvss] search host total %.0f us\n", now_us() - t_start);
  idx->stats.ms_h2d = ms[0];
  idx->stats.ms_encode = ms[1];
  idx->stats.ms_scan = ms[2];
  idx->stats.ms_select = ms[3];
  idx->stats.ms_refine = ms[4];
  idx->stats.ms_topk = ms[5];
  idx->stats.ms_total = tot;
  idx->stats.fixup_sets = fixups;
  unsigned long long hr = 0;
  BVSS_CUDA(cudaMemcpyAsync(&hr, rows, sizeof(hr), cudaMemcpyDeviceToHost, idx->stream));
  BVSS_CUDA(cudaStreamSynchronize(idx->stream));
  idx->stats.cand_rows = hr;
  idx->stats.gather_bytes = hr * static_cast<uint64_t>(idx->dpad) * 2u * (idx->terms == 3 ? 2u : (idx->terms == 1 ? 1u : 0u));
  return BVSS_OK;
}

// ------------------------------------------------------------- sharded --
int bvss_dist_begin(bvss_index* idx, const float* queries, const int64_t* query_offsets, int64_t nq, int32_t k,
                    int32_t T, int64_t id_base, uint32_t flags, bvss_search_ctx** out, int32_t* rounds) {
  if (!out || !rounds) BVSS_FAIL(BVSS_EINVAL, "null out");
  *out = nullptr;
  // (T is the global budget already clamped to the total number of sets, so T < k is legal here when the
  // whole database has fewer than k sets; the caller checks T >= k on its unclamped budget)
  if (T < 1) BVSS_FAIL(BVSS_EINVAL, "T must be >= 1");
  BVSS_TRY(validate_search(idx, queries, query_offsets, nq, k, T < k ? k : T));
  DeviceGuard g(idx->device);
  std::vector<int64_t> qo;
  BVSS_TRY(host_offsets(idx, query_offsets, nq, (flags & BVSS_DEVICE_PTRS) != 0, qo));
  idx->stats = bvss_stats{};
  std::unique_ptr<bvss_search_ctx> c;
  // T is the GLOBAL budget, already clamped by the caller to the total number of sets
  BVSS_TRY(make_ctx(idx, queries, qo, k, T, int64_t(1) << 62, flags, c));
  c->id_base = id_base;
  *rounds = c->rounds;
  *out = c.release();
  return BVSS_OK;
}

int bvss_dist_hist(bvss_search_ctx* c, int32_t round, int32_t* hist_dev) {
  if (!c || !hist_dev) BVSS_FAIL(BVSS_EINVAL, "null argument");
  if (round != c->next_round || round >= c->rounds) BVSS_FAIL(BVSS_ESTATE, "rounds must run in order");
  bvss_index* idx = c->idx;
  DeviceGuard g(idx->device);
  const int key_size = key_size_of(idx);
  BVSS_TRY(launch_select_hist(key_size, c->keys, c->key_stride, idx->n, static_cast<int>(c->nq), c->sel, c->key_bits,
                              round, c->local_hist, idx->stream));
  BVSS_CUDA(cudaMemcpyAsync(hist_dev, c->local_hist, static_cast<size_t>(c->nq) * kHistBins * 4,
                            cudaMemcpyDeviceToDevice, idx->stream));
  return BVSS_OK;
}

int bvss_dist_resolve(bvss_search_ctx* c, int32_t round, const int32_t* global_hist_dev) {
  if (!c || !global_hist_dev) BVSS_FAIL(BVSS_EINVAL, "null argument");
  if (round != c->next_round) BVSS_FAIL(BVSS_ESTATE, "rounds must run in order");
  bvss_index* idx = c->idx;
  DeviceGuard g(idx->device);
  BVSS_TRY(launch_select_resolve(global_hist_dev, c->sel, static_cast<int>(c->nq), c->key_bits, round, idx->stream));
  c->next_round++;
  return BVSS_OK;
}

int bvss_dist_tie_counts(bvss_search_ctx* c, int64_t* eq_dev) {
  if (!c || !eq_dev) BVSS_FAIL(BVSS_EINVAL, "null argument");
  if (c->next_round != c->rounds) BVSS_FAIL(BVSS_ESTATE, "resolve every round first");
  DeviceGuard g(c->idx->device);
  BVSS_TRY(launch_select_tiecount(c->local_hist, c->sel, static_cast<int>(c->nq), eq_dev, c->idx->stream));
  return BVSS_OK;
}

int bvss_dist_finish(bvss_search_ctx* c, const int64_t* all_eq_dev, int32_t world, int32_t rank, int64_t* topk_ids_dev,
                     float* topk_dist_dev) {
  if (!c || !all_eq_dev || !topk_ids_dev || !topk_dist_dev) BVSS_FAIL(BVSS_EINVAL, "null argument");
  if (c->next_round != c->rounds) BVSS_FAIL(BVSS_ESTATE, "resolve every round first");
  if (world < 1 || rank < 0 || rank >= world) BVSS_FAIL(BVSS_EINVAL, "bad rank/world");
  bvss_index* idx = c->idx;
  DeviceGuard g(idx->device);
  BVSS_TRY(launch_select_quota(c->sel, all_eq_dev, static_cast<int>(c->nq), world, rank, idx->stream));
  if (dense_wanted(idx, c->teff / world) && dense_supported(idx, c)) {
    // large global budget: this rank's share of the global top-T as a bitmap over its shard, then the
    // candidate-major refine of the shard (the same kernels as the single-GPU search at this T)
    const int key_size = key_size_of(idx);
    const int64_t words = (idx->n + 31) / 32;
    uint32_t* mask;
    BVSS_TRY(c->alloc(static_cast<size_t>(c->nq) * words * 4, reinterpret_cast<void**>(&mask)));
    BVSS_CUDA(cudaMemsetAsync(mask, 0, static_cast<size_t>(c->nq) * words * 4, idx->stream));
    BVSS_TRY(launch_select_bitmap(key_size, c->keys, c->key_stride, idx->n, static_cast<int>(c->nq), c->sel, c->T,
                                  mask, words, idx->stream, key_limit_of(idx)));
    cudaEventRecord(idx->ev[3], idx->stream);
    bool done = false;
    BVSS_TRY(dense_refine_topk(idx, c, mask, words, -1, topk_ids_dev, topk_dist_dev, &done));
    if (done) return BVSS_OK;
  }
  BVSS_TRY(emit_candidates(idx, c));
  BVSS_TRY(refine_topk(idx, c, topk_ids_dev, topk_dist_dev));
  return BVSS_OK;
}

int bvss_merge_topk(bvss_index* idx, const int64_t* ids_dev, const float* dist_dev, int32_t world, int64_t nq, int32_t k,
                    int64_t* out_ids_dev, float* out_dist_dev) {
  if (!idx || !ids_dev || !dist_dev || !out_ids_dev || !out_dist_dev) BVSS_FAIL(BVSS_EINVAL, "null argument");
  DeviceGuard g(idx->device);
  BVSS_TRY(launch_merge_topk(ids_dev, dist_dev, world, nq, k, out_ids_dev, out_dist_dev, idx->stream));
  return BVSS_OK;
}

void bvss_dist_end(bvss_search_ctx* c) {
  if (!c) return;
  DeviceGuard g(c->idx->device);
  cudaStreamSynchronize(c->idx->stream);
  delete c;
}

}  // extern "C"
