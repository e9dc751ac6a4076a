// group.cu — single-process multi-device index ("Multi-GPU" convention).
//
// A bvss_group owns P shard indexes, shard i on CUDA device devices[i] over the contiguous set-id range
// [base_i, base_{i+1}) (balanced, as dist.py's shard_range).  bvss_group_search runs the exact global-T
// protocol of the sharded search (Alg 6 lines 10-23 with one global candidate budget T) with the
// collectives done inside this process:
//   C1  per radix round: every shard's score histogram is copied to shard 0's device, summed there
//       (sum_hist_kernel) and the global histogram copied back to every shard (all-reduce);
//   C2  every shard's count of keys tied at the global threshold is copied to every shard (all-gather);
//   C3  every shard's local top-k is copied to shard 0 and merged by K7 (bvss_merge_topk).
// The arithmetic of every phase runs in the shard kernels (bvss_dist_*); this file only orders phases and
// moves bytes between devices (cudaMemcpyPeer: NVLink / NVSwitch when peer access is available, staged by
// the driver otherwise).  The heavy phases (encode + scan, refine) of all shards run concurrently, one
// host thread per shard.  A device may hold several shards (devices[] may repeat an ordinal); the result
// is identical for any P and any device assignment (the candidate set is the single-index top-T).
#include <algorithm>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace bvss {

// out[i] = sum over p of in[p][i] (the C1 all-reduce, on shard 0's device)
__global__ void sum_hist_kernel(const int32_t* __restrict__ in, int P, int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t s = 0;
    for (int p = 0; p < P; ++p) s += in[static_cast<int64_t>(p) * n + i];
    out[i] = s;
  }
}

}  // namespace bvss

struct bvss_group {
  std::vector<bvss_index*> shards;
  std::vector<int32_t> dev;   // device of each shard
  std::vector<int64_t> base;  // [P + 1] first global set id of each shard
  int32_t d = 0;
};

namespace {

using bvss::set_error;

// a device buffer freed on scope exit
struct DevBuf {
  void* p = nullptr;
  int dev = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) {
      cudaSetDevice(dev);
      cudaFree(p);
    }
  }
  int alloc(int device, size_t bytes) {
    dev = device;
    BVSS_CUDA(cudaSetDevice(device));
    BVSS_CUDA(cudaMalloc(&p, bytes < 256 ? 256 : bytes));
    return BVSS_OK;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// f(i) for every shard, each on its own host thread; the first failure is returned with its message (the
// library's error text is thread-local) moved to the calling thread
int parallel(int P, const std::function<int(int)>& f) {
  std::vector<int> rc(P, 0);
  std::vector<std::string> msg(P);
  std::vector<std::thread> th;
  th.reserve(P);
  for (int i = 0; i < P; ++i)
    th.emplace_back([&, i] {
      rc[i] = f(i);
      if (rc[i] != BVSS_OK) msg[i] = bvss_last_error();
    });
  for (auto& t : th) t.join();
  for (int i = 0; i < P; ++i)
    if (rc[i] != BVSS_OK) {
      set_error("shard %d: %s", i, msg[i].c_str());
      return rc[i];
    }
  return BVSS_OK;
}

int sync_device(int dev) {
  BVSS_CUDA(cudaSetDevice(dev));
  BVSS_CUDA(cudaDeviceSynchronize());
  return BVSS_OK;
}

void shard_range(int64_t n, int P, int i, int64_t* lo, int64_t* hi) {
  const int64_t b = n / P, r = n % P;
  *lo = i * b + std::min<int64_t>(i, r);
  *hi = *lo + b + (i < r ? 1 : 0);
}

}  // namespace

extern "C" {

int bvss_group_build(const float* vectors, const int64_t* set_offsets, int64_t n, int32_t d, const bvss_params* p,
                     int32_t n_devices, const int32_t* devices, bvss_group** out) {
  if (!out) BVSS_FAIL(BVSS_EINVAL, "null out");
  *out = nullptr;
  if (!vectors || !set_offsets || !p) BVSS_FAIL(BVSS_EINVAL, "null argument");
  if (p->flags & BVSS_DEVICE_PTRS) BVSS_FAIL(BVSS_EINVAL, "bvss_group_build takes host arrays");
  if (n < 1) BVSS_FAIL(BVSS_EINVAL, "n must be >= 1");
  if (n_devices == -1) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess || c < 1)
      BVSS_FAIL(BVSS_EUNSUPPORTED, "no CUDA device available (no CPU fallback)");
    n_devices = c;
  }
  if (n_devices < 1 || n_devices > 64) BVSS_FAIL(BVSS_EINVAL, "n_devices must be -1 or 1..64");
  if (set_offsets[0] != 0) BVSS_FAIL(BVSS_EINVAL, "offsets must start at 0");
  for (int64_t i = 0; i < n; ++i)
    if (set_offsets[i + 1] <= set_offsets[i])
      BVSS_FAIL(BVSS_EINVAL, "set %lld is empty or offsets decrease (Def 2: m >= 1)", static_cast<long long>(i));
  const int P = static_cast<int>(std::min<int64_t>(n_devices, n));
  std::unique_ptr<bvss_group> g(new bvss_group());
  g->d = d;
  g->shards.assign(P, nullptr);
  g->dev.resize(P);
  g->base.resize(P + 1);
  std::vector<std::vector<int64_t>> sub(P);
  for (int i = 0; i < P; ++i) {
    int64_t lo, hi;
    shard_range(n, P, i, &lo, &hi);
    g->base[i] = lo;
    g->dev[i] = devices ? devices[i] : i;
    sub[i].resize(hi - lo + 1);
    for (int64_t j = lo; j <= hi; ++j) sub[i][j - lo] = set_offsets[j] - set_offsets[lo];
  }
  g->base[P] = n;
  const int rc = parallel(P, [&](int i) {
    bvss_params q = *p;
    q.device = g->dev[i];
    const int64_t lo = g->base[i], hi = g->base[i + 1];
    return bvss_build_index(vectors + set_offsets[lo] * static_cast<int64_t>(d), sub[i].data(), hi - lo, d, &q,
                            &g->shards[i]);
  });
  if (rc != BVSS_OK) {
    for (bvss_index* s : g->shards) bvss_free_index(s);
    return rc;
  }
  *out = g.release();
  return BVSS_OK;
}

int bvss_group_search(bvss_group* g, const float* queries, const int64_t* query_offsets, int64_t nq, int32_t k,
                      int32_t T, int64_t* out_ids, float* out_dist, uint32_t flags) {
  if (!g || !queries || !query_offsets || !out_ids || !out_dist) BVSS_FAIL(BVSS_EINVAL, "null argument");
  if (flags & BVSS_DEVICE_PTRS) BVSS_FAIL(BVSS_EINVAL, "bvss_group_search takes host arrays");
  const int P = static_cast<int>(g->shards.size());
  if (P == 1) return bvss_search(g->shards[0], queries, query_offsets, nq, k, T, out_ids, out_dist, flags);
  if (nq < 1 || k < 1) BVSS_FAIL(BVSS_EINVAL, "nq and k must be >= 1");
  if (T < k) BVSS_FAIL(BVSS_EINVAL, "T (%d) < k (%d) (reading R16)", T, k);
  const int64_t n = g->base[P];
  const int32_t Teff = static_cast<int32_t>(std::min<int64_t>(T, n));  // T > n: brute force over all sets
  std::vector<bvss_search_ctx*> ctx(P, nullptr);
  std::vector<int32_t> rounds(P, 0);
  struct Ends {  // every context is ended on every exit path
    std::vector<bvss_search_ctx*>& c;
    ~Ends() {
      for (auto* x : c) bvss_dist_end(x);
    }
  } ends{ctx};
  BVSS_TRY(parallel(P, [&](int i) {
    return bvss_dist_begin(g->shards[i], queries, query_offsets, nq, k, Teff, g->base[i], flags, &ctx[i], &rounds[i]);
  }));
  for (int i = 1; i < P; ++i)
    if (rounds[i] != rounds[0]) BVSS_FAIL(BVSS_ESTATE, "shards disagree on the radix rounds");
  const size_t hbytes = static_cast<size_t>(nq) * 2048 * 4, kk = static_cast<size_t>(nq) * k;
  std::vector<DevBuf> hist(P), ghist(P), eq(P), alleq(P), tids(P), td(P);
  DevBuf stage, all_ids, all_d, oid, od;
  for (int i = 0; i < P; ++i) {
    BVSS_TRY(hist[i].alloc(g->dev[i], hbytes));
    BVSS_TRY(ghist[i].alloc(g->dev[i], hbytes));
    BVSS_TRY(eq[i].alloc(g->dev[i], nq * 8));
    BVSS_TRY(alleq[i].alloc(g->dev[i], static_cast<size_t>(P) * nq * 8));
    BVSS_TRY(tids[i].alloc(g->dev[i], kk * 8));
    BVSS_TRY(td[i].alloc(g->dev[i], kk * 4));
  }
  const int d0 = g->dev[0];
  BVSS_TRY(stage.alloc(d0, hbytes * P));
  BVSS_TRY(all_ids.alloc(d0, kk * 8 * P));
  BVSS_TRY(all_d.alloc(d0, kk * 4 * P));
  BVSS_TRY(oid.alloc(d0, kk * 8));
  BVSS_TRY(od.alloc(d0, kk * 4));
  for (int r = 0; r < rounds[0]; ++r) {  // C1: all-reduce of the round's histograms
    for (int i = 0; i < P; ++i) BVSS_TRY(bvss_dist_hist(ctx[i], r, hist[i].as<int32_t>()));
    for (int i = 0; i < P; ++i) BVSS_TRY(sync_device(g->dev[i]));
    for (int i = 0; i < P; ++i)
      BVSS_CUDA(cudaMemcpyPeer(stage.as<uint8_t>() + i * hbytes, d0, hist[i].p, g->dev[i], hbytes));
    BVSS_CUDA(cudaSetDevice(d0));
    bvss::sum_hist_kernel<<<256, 256>>>(stage.as<int32_t>(), P, static_cast<int64_t>(nq) * 2048,
                                        ghist[0].as<int32_t>());
    BVSS_CUDA(cudaGetLastError());
    BVSS_TRY(sync_device(d0));
    for (int i = 1; i < P; ++i) BVSS_CUDA(cudaMemcpyPeer(ghist[i].p, g->dev[i], ghist[0].p, d0, hbytes));
    for (int i = 0; i < P; ++i) BVSS_TRY(sync_device(g->dev[i]));
    for (int i = 0; i < P; ++i) BVSS_TRY(bvss_dist_resolve(ctx[i], r, ghist[i].as<int32_t>()));
  }
  // C2: all-gather of the tie counts
  for (int i = 0; i < P; ++i) BVSS_TRY(bvss_dist_tie_counts(ctx[i], eq[i].as<int64_t>()));
  for (int i = 0; i < P; ++i) BVSS_TRY(sync_device(g->dev[i]));
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j)
      BVSS_CUDA(cudaMemcpyPeer(alleq[i].as<int64_t>() + static_cast<size_t>(j) * nq, g->dev[i], eq[j].p, g->dev[j],
                               nq * 8));
  for (int i = 0; i < P; ++i) BVSS_TRY(sync_device(g->dev[i]));
  // each shard's share of the global top-T, refined concurrently
  BVSS_TRY(parallel(P, [&](int i) {
    BVSS_TRY(bvss_dist_finish(ctx[i], alleq[i].as<int64_t>(), P, i, tids[i].as<int64_t>(), td[i].as<float>()));
    return sync_device(g->dev[i]);
  }));
  // C3 + K7
  for (int i = 0; i < P; ++i) {
    BVSS_CUDA(cudaMemcpyPeer(all_ids.as<int64_t>() + i * kk, d0, tids[i].p, g->dev[i], kk * 8));
    BVSS_CUDA(cudaMemcpyPeer(all_d.as<float>() + i * kk, d0, td[i].p, g->dev[i], kk * 4));
  }
  BVSS_TRY(sync_device(d0));
  BVSS_TRY(bvss_merge_topk(g->shards[0], all_ids.as<int64_t>(), all_d.as<float>(), P, nq, k, oid.as<int64_t>(),
                           od.as<float>()));
  BVSS_TRY(sync_device(d0));
  BVSS_CUDA(cudaMemcpy(out_ids, oid.p, kk * 8, cudaMemcpyDeviceToHost));
  BVSS_CUDA(cudaMemcpy(out_dist, od.p, kk * 4, cudaMemcpyDeviceToHost));
  return BVSS_OK;
}

int32_t bvss_group_shards(const bvss_group* g) { return g ? static_cast<int32_t>(g->shards.size()) : 0; }

int bvss_group_shard(const bvss_group* g, int32_t shard, bvss_index** out, int64_t* id_base) {
  if (!g || !out || shard < 0 || shard >= static_cast<int32_t>(g->shards.size()))
    BVSS_FAIL(BVSS_EINVAL, "bad group or shard");
  *out = g->shards[shard];
  if (id_base) *id_base = g->base[shard];
  return BVSS_OK;
}

void bvss_free_group(bvss_group* g) {
  if (!g) return;
  for (bvss_index* s : g->shards) bvss_free_index(s);
  delete g;
}

}  // extern "C"
