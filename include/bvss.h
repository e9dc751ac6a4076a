/*
 * bvss.h — C ABI of the B200-native BioVSS hot path (arXiv 2412.03301).
 *
 * The library (paper_2412_03301_b200/libbvss.so) implements top-k vector-set
 * search under the Hausdorff distance (Def 4), filtered by
 * FlyHash codes (Def 7; Alg 1) folded into per-set Bloom
 * or count-Bloom sketches (Def 10 P:729-732 / Alg 5; Def 8 P:657 / Alg 3), with
 * the cascade of Alg 6 run with stage 1 open (reading R6):
 * sketch scan -> top-T candidates -> exact Hausdorff rerank -> top-k.
 *
 * Every step runs in hand-written sm_100a kernels.  There is no CPU fallback:
 * on a machine without an sm_100 device every compute entry point returns
 * BVSS_EUNSUPPORTED (or BVSS_ECUDA) and sets bvss_last_error().
 *
 * Conventions (all entry points):
 *  - Return 0 (BVSS_OK) on success or a negative bvss_status; never throw,
 *    never abort.  A thread-local message describes the last failure.
 *  - Ownership: inputs are caller-owned; the library copies what it keeps
 *    before returning and never retains caller pointers.  Outputs are
 *    caller-allocated.  An index owns all of its device memory until
 *    bvss_free_index().
 *  - Pointers are HOST pointers unless BVSS_DEVICE_PTRS is passed in the call's
 *    flags, in which case every array argument of that call is a device
 *    pointer on the index's device.  Host inputs may be pageable or pinned.
 *  - Set ids are positions 0..n-1 in set_offsets (int64).  Vectors are fp32,
 *    row-major [rows][d].  set_offsets[0] == 0, strictly increasing (Def 2:
 *    every set has m >= 1 vectors), set_offsets[n] == number of rows.
 *  - Bits: code/sketch Bloom position j lives in uint32 word j>>5, bit j&31.
 *  - Results are sorted by (distance ascending, id ascending); missing
 *    results (k > n) are padded with id -1 and distance +inf.
 *  - An index is not thread-safe; distinct indexes are independent.
 *  - All work of a call is issued on the index's stream (bvss_set_stream);
 *    calls with host outputs synchronise that stream before returning; calls
 *    with BVSS_DEVICE_PTRS are asynchronous with respect to the host.
 */
#ifndef BVSS_H
#define BVSS_H

#include <stdint.h>

#if defined(__GNUC__)
#define BVSS_API __attribute__((visibility("default")))
#else
#define BVSS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BVSS_OK = 0,
  BVSS_EINVAL = -1,       /* bad argument (null, sizes, offsets, L>m, s>d, m%32, k<1, T<k, ...) */
  BVSS_ENONFINITE = -2,   /* NaN/Inf found while BVSS_VALIDATE_FINITE was set */
  BVSS_ENOMEM = -3,       /* device or host allocation failed */
  BVSS_ECUDA = -4,        /* a CUDA runtime error (message has the CUDA error string) */
  BVSS_EUNSUPPORTED = -5, /* no sm_100 device, or a size beyond this build's limits */
  BVSS_ESTATE = -6,       /* call out of order (e.g. distributed phases) */
  BVSS_ENCCL = -7         /* reserved for a collective failure; the sharded phases below leave the collectives
                             to the caller (torch.distributed / NCCL), whose errors surface there */
} bvss_status;

typedef enum { BVSS_SKETCH_BINARY = 0, BVSS_SKETCH_COUNT_U8 = 1 } bvss_sketch_kind;

/* call flags */
#define BVSS_DEVICE_PTRS 0x1u      /* array arguments are device pointers */
#define BVSS_VALIDATE_FINITE 0x2u  /* reject NaN/Inf inputs (one extra pass) */
#define BVSS_KEEP_CODES 0x4u       /* build: keep per-vector codes for bvss_export_codes */

typedef struct {
  uint32_t m;            /* code length b = Bloom length (reading R21); m % 32 == 0, 32 <= m <= 2048 */
  uint32_t s;            /* ones per projection row, 1 <= s <= min(d, 32) */
  uint32_t L;            /* WTA winners L_wta, 1 <= L <= m */
  uint32_t sketch;       /* bvss_sketch_kind */
  uint64_t seed;         /* projection seed (reading R7) */
  const uint16_t* projection; /* optional host [m][s] sorted row indices; NULL = generate from seed */
  int32_t device;        /* CUDA device ordinal of this index (shard) */
  uint32_t flags;        /* build flags (BVSS_DEVICE_PTRS | BVSS_VALIDATE_FINITE | BVSS_KEEP_CODES) */
  uint32_t query_batch;  /* queries per internal sub-batch; 0 = auto */
  uint32_t refine_terms; /* tensor-core Gram on the scaled fp16 split: 0 = default (= 1), 1 = hi*hi,
                            3 = hi*hi + hi*lo + lo*hi, 255 = no tensor pass (exact fp32 for every candidate) */
  uint32_t select_mode;  /* bvss_search candidate selection: 0 = auto, 1 = full key rows (scan writes every
                            score, radix select over them), 2 = sampled threshold (scan emits only scores <=
                            a per-query threshold estimated on a database sample; exact, with a per-batch
                            fallback to 1 when the estimate is too low or the buffer overflows).  Auto = 2 for
                            binary sketches when the tensor-core scan runs and n >= 65536 (count-sketch keys
                            tie massively at the threshold).  Results are identical. */
  uint32_t metric;       /* rerank distance (bvss_metric): 0 = Hausdorff (Def 4; the paper's
                            metric), 1 = MeanMin d_mean-min(Q, V) = 1/|Q| sum_q min_v ||q - v|| (the
                            query set first, reading R23), 2 = Min d_min(Q, V) = min ||q - v||.
                            The §3.2 alternatives; the filter is unchanged. */
  uint32_t score;        /* filter score (bvss_score_kind): 0 = Hamming (binary) / squared L2 (count,
                            reading R2); 1 = OVERLAP (reading R24): rank by the shared-bit count
                            popc(S_Q AND S_i) (count: the dot product <C_Q, C_i>) descending, ties by id;
                            bvss_filter reports it as the ascending key 2 (m - popc) (binary) /
                            2 (m 255^2 - dot) (count); 2 = BINARIZED (reading R25): Hamming between
                            the binarised counters (C_Q > 0) and (C_i > 0), which equal the OR-fold
                            binary sketches, so a count index scored BINARIZED is built as a binary
                            index (bvss_get_info / bvss_export_sketches then report binary sketches);
                            3 = L1 (reading R26): sum_j |C_Q[j] - C_i[j]| for count sketches (SIMT
                            vabsdiffu4 / dp4a scan, full-key select); on binary sketches L1 = Hamming. */
  uint32_t gate_A;       /* BioVSS++ stage 1 (Alg 6 lines 1, 3-9; the inverted index of Alg 4):
                            the query's count Bloom filter picks its gate_A largest positions P (ties -> lower
                            position, reading R27) and only sets with C_i[p] >= gate_M for some p in P are
                            candidates; 0 = stage 1 open (F1 = D, reading R6); at most min(64, m).  The paper's
                            defaults are A = 3, M = 1.  A binary-sketch index supports gate_M <= 1
                            (S = (C > 0)).  Candidates are then the first T of F1 by (score, id); |F1| < T
                            returns F1 whole (bvss_filter pads with -1). */
  uint32_t gate_M;       /* the gate's minimum count M (0 = open) */
  uint32_t filter;       /* candidate generation: 0 = the sketch scan of Alg 6 (default); 1 = BioVSS Alg 2
                            (P:363-390): Haus^H(Q^H, H_j), the Hausdorff aggregation of Hamming distances
                            between per-vector codes, ranks every set and the c = T smallest
                            (ties by id) are refined; the index keeps its codes.  bvss_filter reports Haus^H
                            as the score. */
} bvss_params;

typedef enum { BVSS_SCORE_DEFAULT = 0, BVSS_SCORE_OVERLAP = 1, BVSS_SCORE_BINARIZED = 2, BVSS_SCORE_L1 = 3 } bvss_score_kind;

typedef enum { BVSS_METRIC_HAUSDORFF = 0, BVSS_METRIC_MEANMIN = 1, BVSS_METRIC_MIN = 2 } bvss_metric;

typedef struct bvss_index bvss_index;

typedef struct {
  int64_t n, nvec;       /* sets and vectors in the index */
  int32_t d, dpad;       /* dimension, and its padding to a multiple of 64 for the fp16 copies */
  uint32_t m, s, L, sketch;
  int32_t device;
  uint64_t device_bytes; /* device memory owned by the index (excluding search workspace) */
  uint64_t workspace_bytes;
} bvss_info;

typedef struct {
  /* per-stage device time of the most recent bvss_search / bvss_filter / bvss_refine, ms */
  float ms_h2d, ms_encode, ms_scan, ms_select, ms_refine, ms_topk, ms_d2h, ms_total;
  uint64_t scan_bytes;    /* database-operand bytes the scan kernel streams (FP4/u8 tiles; algorithmic) */
  uint64_t gather_bytes;  /* candidate-vector bytes gathered by the refine kernel (algorithmic) */
  uint64_t cand_rows;     /* candidate vectors refined */
  uint64_t fixup_sets;    /* candidates recomputed by the exact fp32 fix-up */
  int32_t kernel_launches;/* kernels launched by the call */
  int32_t query_batch;
  uint64_t select_batches;   /* query batches selected on the sampled-threshold path */
  uint64_t select_fallbacks; /* of those, batches redone on the full-key path */
  uint64_t scan_macs;        /* (query sketch bit, database sketch bit) products of the scan (nq x n x m) */
  /* candidate-major (dense) refine: batches it ran, (query set, database set) pairs that
     survived the lower-bound prune, candidates it emitted to the exact top-k, (query vector, database vector)
     pairs and tensor-core flop (2 x M x N x K of every MMA tile, padding included) */
  uint64_t dense_batches, dense_survivors, dense_emitted, dense_pairs;
  double dense_flop;
} bvss_stats;

/* ---------------------------------------------------------------- core -- */

/* Build an index over n sets (Alg 1 + Alg 3 / Alg 5, P:323-343, P:665-682,
 * P:738-757): copies vectors to the device, generates W (or takes p->projection),
 * encodes every vector (FlyHash + WTA), folds per-set sketches, and prepares the
 * refine operands (fp16 hi/lo split, fp32 squared norms).
 *   vectors     [set_offsets[n]][d] fp32
 *   set_offsets [n+1] int64
 * Errors: BVSS_EINVAL for bad sizes/offsets/params, BVSS_ENONFINITE (with
 * BVSS_VALIDATE_FINITE), BVSS_ENOMEM, BVSS_ECUDA, BVSS_EUNSUPPORTED. */
BVSS_API int bvss_build_index(const float* vectors, const int64_t* set_offsets, int64_t n, int32_t d,
                     const bvss_params* p, bvss_index** out);

/* Approximate top-k vector-set search (Def 5 P:162-169 via Alg 6):
 * for each query set, scan all n sketches, keep the T smallest filter scores
 * (ties -> lower id), rerank them by exact Hausdorff distance, return the k
 * nearest.  T >= n gives exact brute force.  T is clamped to n.
 *   queries       [query_offsets[nq]][d] fp32
 *   query_offsets [nq+1] int64
 *   out_ids  [nq][k] int64, out_dist [nq][k] fp32 (Hausdorff distance, not squared)
 * Errors: BVSS_EINVAL (k < 1, T < k, bad offsets), plus the build errors. */
BVSS_API int bvss_search(bvss_index* idx, const float* queries, const int64_t* query_offsets, int64_t nq,
                int32_t k, int32_t T, int64_t* out_ids, float* out_dist, uint32_t flags);

/* Streaming build, for databases larger than host memory (cfg5 is 98 GB): declare the
 * totals, append sets in order in chunks (vectors [local_offsets[n_chunk]][d] fp32 and local_offsets
 * [n_chunk+1] starting at 0, host pointers unless p->flags has BVSS_DEVICE_PTRS; the chunk buffers may
 * be reused when append returns), then finish, which runs the build of bvss_build_index on the
 * appended data (identical result).  Until finish every search call returns BVSS_ESTATE.
 * Errors: BVSS_EINVAL (sizes, offsets, more data than declared, finish before all of it arrived),
 * BVSS_ESTATE (append/finish on a finished index), plus the build errors. */
BVSS_API int bvss_index_begin(int64_t n_total, int64_t nvec_total, int32_t d, const bvss_params* p,
                     bvss_index** out);
BVSS_API int bvss_index_append(bvss_index* idx, const float* vectors, const int64_t* local_offsets,
                      int64_t n_chunk);
BVSS_API int bvss_index_finish(bvss_index* idx);

BVSS_API void bvss_free_index(bvss_index* idx);
BVSS_API const char* bvss_last_error(void);
BVSS_API int bvss_get_info(const bvss_index* idx, bvss_info* out);
BVSS_API int bvss_get_stats(const bvss_index* idx, bvss_stats* out);
/* Issue all work of this index on `stream` (a cudaStream_t; NULL = the index's own non-blocking
 * stream, which is NOT ordered with the legacy default stream: pass cudaStreamLegacy to use that). */
BVSS_API int bvss_set_stream(bvss_index* idx, void* stream);
/* Number of sm_100-class devices visible (0 if none); never fails. */
BVSS_API int bvss_device_count(void);

/* ---------------------------------------------------- stage entry points -- */

/* W as built, host [m][s] uint16 (a-1). */
BVSS_API int bvss_export_projection(const bvss_index* idx, uint16_t* out);
/* Codes of vectors [first, first+count), host [count][m/32] uint32 (a-2).
 * Needs BVSS_KEEP_CODES at build. */
BVSS_API int bvss_export_codes(const bvss_index* idx, int64_t first, int64_t count, uint32_t* out);
/* Sketches of sets [first, first+count) in row-major host layout (a-3):
 * binary: uint32 [count][m/32]; count-Bloom: uint8 [count][m]. */
BVSS_API int bvss_export_sketches(const bvss_index* idx, int64_t first, int64_t count, void* out);
/* Query sketches (a-4: Alg 6 lines 1-2), same layout as above,
 * host [nq][m/32] uint32 or [nq][m] uint8; codes optional ([rows][m/32], may be NULL). */
BVSS_API int bvss_query_sketch(bvss_index* idx, const float* queries, const int64_t* query_offsets, int64_t nq,
                      void* out_sketch, uint32_t* out_codes, uint32_t flags);
/* Filter (a-5 + a-6: Alg 6 lines 10-18): per query the min(T, n) candidates in
 * ASCENDING id order and their filter scores (binary: Hamming; count: squared
 * L2 between counters, reading R2).  out_cand [nq][T] int32 (padded with -1),
 * out_score [nq][T] int32 (may be NULL). */
BVSS_API int bvss_filter(bvss_index* idx, const float* queries, const int64_t* query_offsets, int64_t nq,
                int32_t T, int32_t* out_cand, int32_t* out_score, uint32_t flags);
/* Refine (a-7 + a-8: Alg 6 lines 19-23): given candidate lists (as from
 * bvss_filter, -1 padded), compute the tensor-core Hausdorff of every candidate
 * and the exact top-k.  out_approx [nq][T] fp32 receives the tensor-core
 * value per candidate (NaN where cand == -1; may be NULL): the squared
 * distance for Hausdorff and Min, the distance for MeanMin (bvss_params.metric). */
BVSS_API int bvss_refine(bvss_index* idx, const float* queries, const int64_t* query_offsets, int64_t nq,
                const int32_t* cand, int32_t T, int32_t k, int64_t* out_ids, float* out_dist,
                float* out_approx, uint32_t flags);
/* Brute force (K8; "precise calculations according to Definition 4"):
 * the exact top-k Hausdorff neighbours among sets [0, set_limit) (set_limit
 * <= 0 or > n means all n sets), for recall ground truth.  Runs the refine
 * path (tensor-core Hausdorff + exact fp32 fix-up window, exact by the window
 * rule) over chunks of 8192 sets and merges the chunk top-k lists (K7).
 *   out_ids [nq][k] int64, out_dist [nq][k] fp32, sorted by (distance, id),
 *   padded with (-1, +inf) when set_limit < k.
 * Errors: as bvss_search. */
BVSS_API int bvss_bruteforce(bvss_index* idx, const float* queries, const int64_t* query_offsets, int64_t nq,
                    int64_t set_limit, int32_t k, int64_t* out_ids, float* out_dist, uint32_t flags);
/* Squared-distance error bound E used by the fix-up window for a query whose
 * largest vector norm is qnorm_max. */
BVSS_API double bvss_refine_error_bound(const bvss_index* idx, double qnorm_max);

/* ------------------------------------------- sharded (multi-GPU) search -- */
/* Exact global-T protocol over P shards: each rank holds an
 * index over a contiguous id range [id_base, id_base + n).  The caller runs
 * the collectives (NCCL via torch.distributed) between phases; all buffers
 * named *_dev are device pointers on the index's device.                     */
typedef struct bvss_search_ctx bvss_search_ctx;

/* Encode + sketch + scan one query batch; returns the number of radix rounds.
 * T is the GLOBAL candidate budget already clamped to the total number of
 * sets (it may then be < k; the caller rejects an unclamped T < k).        */
BVSS_API int bvss_dist_begin(bvss_index* idx, const float* queries, const int64_t* query_offsets, int64_t nq,
                    int32_t k, int32_t T, int64_t id_base, uint32_t flags, bvss_search_ctx** out,
                    int32_t* rounds);
/* Local histogram of radix round r: hist_dev int32 [nq][2048]. */
BVSS_API int bvss_dist_hist(bvss_search_ctx* ctx, int32_t round, int32_t* hist_dev);
/* Apply the GLOBAL (all-reduced) histogram of round r. */
BVSS_API int bvss_dist_resolve(bvss_search_ctx* ctx, int32_t round, const int32_t* global_hist_dev);
/* Local count of candidates tied at the global threshold: eq_dev int64 [nq]. */
BVSS_API int bvss_dist_tie_counts(bvss_search_ctx* ctx, int64_t* eq_dev);
/* Given the all-gathered tie counts [P][nq] int64 of every rank, take this
 * rank's share of the global top-T, refine it and write the local top-k
 * (global ids) to topk_ids_dev [nq][k] int64 and topk_dist_dev [nq][k] fp32. */
BVSS_API int bvss_dist_finish(bvss_search_ctx* ctx, const int64_t* all_eq_dev, int32_t world, int32_t rank,
                     int64_t* topk_ids_dev, float* topk_dist_dev);
/* Merge P local top-k lists [P][nq][k] into the global top-k [nq][k] (K7). */
BVSS_API int bvss_merge_topk(bvss_index* idx, const int64_t* ids_dev, const float* dist_dev, int32_t world,
                    int64_t nq, int32_t k, int64_t* out_ids_dev, float* out_dist_dev);
BVSS_API void bvss_dist_end(bvss_search_ctx* ctx);

/* -------------------------------- single-process multi-device index -- */
/* SURVEY §8(b) "Multi-GPU" convention without torch.distributed: one process
 * drives P shard indexes, shard i on CUDA device devices[i] (NULL: 0..P-1; an
 * ordinal may repeat, several shards then share a device) over the contiguous,
 * balanced set-id range [base_i, base_{i+1}) of the database.  Search runs the
 * exact global-T protocol above (Alg 6 lines 10-23, P:795-814,
 * with ONE global candidate budget T) with the collectives in-process: score
 * histograms summed on shard 0's device and copied back (C1), tie counts
 * all-gathered (C2), local top-k lists merged by K7 on shard 0 (C3), the bytes
 * moved by cudaMemcpyPeer (NVLink / NVSwitch where peer access exists).  The
 * encode + scan and refine phases of all shards run concurrently (one host
 * thread per shard).  Results are identical to one index over the whole
 * database, for any P and device assignment.                               */
typedef struct bvss_group bvss_group;

/* Build a group over n sets: n_devices = P in 1..64, or -1 = every visible
 * device; P is reduced to n when n < P.  vectors / set_offsets are HOST arrays
 * (BVSS_DEVICE_PTRS in p->flags is EINVAL); p->device is ignored (devices[]
 * decides).  Each shard is built as by bvss_build_index (same params, same
 * projection W), concurrently.  Errors: EINVAL as bvss_build_index plus a
 * bad n_devices; a shard's failure frees the shards built so far and returns
 * its status with the message prefixed "shard i:".                         */
BVSS_API int bvss_group_build(const float* vectors, const int64_t* set_offsets, int64_t n, int32_t d,
                              const bvss_params* p, int32_t n_devices, const int32_t* devices, bvss_group** out);
/* Exact top-k of nq query sets (HOST arrays; flags may carry
 * BVSS_VALIDATE_FINITE), out_ids [nq][k] int64 global set ids, out_dist
 * [nq][k] fp32, as bvss_search.  P = 1 is bvss_search on the only shard. */
BVSS_API int bvss_group_search(bvss_group* g, const float* queries, const int64_t* query_offsets, int64_t nq,
                               int32_t k, int32_t T, int64_t* out_ids, float* out_dist, uint32_t flags);
/* Number of shards (0 for NULL). */
BVSS_API int32_t bvss_group_shards(const bvss_group* g);
/* Shard i's index (owned by the group: do not free it) and its first global
 * set id (for bvss_get_stats / bvss_get_info / exports).                   */
BVSS_API int bvss_group_shard(const bvss_group* g, int32_t shard, bvss_index** out, int64_t* id_base);
BVSS_API void bvss_free_group(bvss_group* g);

#ifdef __cplusplus
}
#endif
#endif /* BVSS_H */
