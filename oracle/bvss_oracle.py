"""Plain CPU oracle for the BioVSS hot path (arXiv 2412.03301).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module. The product path (``paper_2412_03301_b200``) never imports it, and this
module imports nothing from the product path: the two share no code, headers,
tables or constants. Only the seeded input generator (``gen/synth.py``, which
holds none of the method's arithmetic) feeds both.

Every function follows one passage of ``PAPER.md`` (cited as ``P:<line>``,
plus the definition / algorithm it falls in) in the paper's order and notation,
or, where the paper is silent, the reading recorded in ``DESIGN.md`` §3
(cited as ``R<n>``). Floating point is fp64 except where a reading fixes fp32
(the FlyHash activations, R8, so that codes can be compared bit for bit).

Parity status of each function is stated in its docstring; the pins live in
``tests/test_oracle_*.py`` and ``tests/golden/``. Recall on synthetic data is
*parity unpinned* (the paper's recalls were measured on datasets that are not
available here).

Bit convention (R21): code / sketch bit ``j`` (0-based Bloom position) lives in
``uint32`` word ``j >> 5``, bit ``j & 31``.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1

# ---------------------------------------------------------------------------
# a-1: the projection W  (Def 7; reading R7)
# ---------------------------------------------------------------------------


def splitmix64_stream(state: int):
    """SplitMix64 (Steele/Lea/Flood; Vigna's reference constants), as a Python
    generator over unbounded ints reduced mod 2**64.  Reading R7 fixes this RNG
    so that two independent implementations of W agree.  Pinned by the
    published known-answer values for state 0 (tests/golden/splitmix64.json)."""
    x = state & MASK64
    while True:
        x = (x + 0x9E3779B97F4A7C15) & MASK64
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        yield z ^ (z >> 31)


def projection(seed: int, m: int, s: int, d: int) -> np.ndarray:
    """FlyHash projection W in {0,1}^{m x d} with exactly ``s`` ones per row
    (Def 7: "W in R^{b x d} is a random projection matrix"; BJ cfg1:
    "each projection row has 6 ones at uniformly sampled input dims").

    Returned in index form: uint16 ``[m][s]``, row j = the sorted column
    indices of the ones in row j.  Reading R7: row j draws from SplitMix64
    seeded with ``seed ^ (j * 0xD1B54A32D192ED03)``; a draw ``u`` is rejected
    when ``r = 2**64 mod d`` is non-zero and ``u >= 2**64 - r`` (no modulo
    bias), else ``i = u mod d`` is taken unless already chosen.
    """
    if not (1 <= s <= d):
        raise ValueError("need 1 <= s <= d")
    if d > 65535:
        raise ValueError("d must fit uint16")
    W = np.zeros((m, s), dtype=np.uint16)
    r = (1 << 64) % d
    for j in range(m):
        rng = splitmix64_stream(seed ^ ((j * 0xD1B54A32D192ED03) & MASK64))
        chosen: list[int] = []
        while len(chosen) < s:
            u = next(rng)
            if r != 0 and u >= (1 << 64) - r:
                continue
            i = u % d
            if i not in chosen:
                chosen.append(i)
        W[j] = sorted(chosen)
    return W


# ---------------------------------------------------------------------------
# a-2: FlyHash activations + WTA  (Def 7, Alg 1)
# ---------------------------------------------------------------------------


def activations(V: np.ndarray, W: np.ndarray) -> np.ndarray:
    """h_p = W v for every row v of V (Alg 1 line 5, "Matrix projection").

    W is binary, so (W v)_j = sum_{i in S_j} v_i.  Reading R8 fixes the fp32
    summation order: start from +0.0f and add v[S_j[0]], v[S_j[1]], ... left to
    right, each addition rounded to nearest even in fp32 (no FMA, no pairwise
    summation).  Returns fp32 ``[N][m]``.
    """
    V = np.ascontiguousarray(V, dtype=np.float32)
    N = V.shape[0]
    m, s = W.shape
    acc = np.zeros((N, m), dtype=np.float32)
    for t in range(s):
        # one fp32 addition per step, elementwise: acc_j <- fl(acc_j + v[W[j,t]])
        acc = acc + V[:, W[:, t].astype(np.int64)]
    return acc


def activations_fp64(V: np.ndarray, W: np.ndarray) -> np.ndarray:
    """The same projection in fp64 (used only to classify near-ties, the
    BJ north_star exemption: |a_(L) - a_(L+1)| < 1e-5 |a_(L)|)."""
    V = np.asarray(V, dtype=np.float64)
    m, s = W.shape
    acc = np.zeros((V.shape[0], m), dtype=np.float64)
    for t in range(s):
        acc = acc + V[:, W[:, t].astype(np.int64)]
    return acc


def wta(a: np.ndarray, L: int) -> np.ndarray:
    """Winner-take-all (Def 7): set the L largest entries to 1, the rest
    to 0, so ||h||_1 = L exactly.  Reading R4: among equal activations the
    lower row index wins.  Returns bool ``[N][m]``."""
    N, m = a.shape
    if not (1 <= L <= m):
        raise ValueError("need 1 <= L <= m")
    # stable sort of -a keeps ascending j among equal values; +0.0 folds -0.0
    order = np.argsort(-(a + np.float32(0.0)), axis=1, kind="stable")[:, :L]
    h = np.zeros((N, m), dtype=bool)
    np.put_along_axis(h, order, True, axis=1)
    return h


def pack_bits(h: np.ndarray) -> np.ndarray:
    """bool ``[N][m]`` -> uint32 ``[N][m/32]`` with bit j in word j>>5, bit j&31."""
    N, m = h.shape
    if m % 32:
        raise ValueError("m must be a multiple of 32")
    b = h.reshape(N, m // 32, 32).astype(np.uint64)
    weights = (np.uint64(1) << np.arange(32, dtype=np.uint64))
    return (b * weights).sum(axis=2).astype(np.uint32)


def unpack_bits(words: np.ndarray, m: int) -> np.ndarray:
    """uint32 ``[N][m/32]`` -> bool ``[N][m]`` (inverse of pack_bits)."""
    w = np.asarray(words, dtype=np.uint32)
    bits = (w[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1
    return bits.reshape(w.shape[0], m).astype(bool)


def encode(V: np.ndarray, W: np.ndarray, L: int, chunk: int = 8192) -> np.ndarray:
    """Gen_Binary_Codes (Alg 1) for a flat array of vectors: the
    packed code h = WTA(W v, L) of every row.  Returns uint32 ``[N][m/32]``."""
    out = []
    for i in range(0, V.shape[0], chunk):
        out.append(pack_bits(wta(activations(V[i:i + chunk], W), L)))
    if not out:
        return np.zeros((0, W.shape[0] // 32), dtype=np.uint32)
    return np.concatenate(out, axis=0)


def near_tie_rows(V: np.ndarray, W: np.ndarray, L: int, rel: float = 1e-5) -> np.ndarray:
    """Rows j whose fp64 activation lies within rel*|a_(L)| of the L-th largest
    activation a_(L): the only rows where a GPU code may legitimately differ
    (BJ north_star: "Codes are bit-exact except where the L-th and (L+1)-th
    activations differ by <1e-5 relative").  Returns bool ``[N][m]``."""
    a = activations_fp64(V, W)
    srt = -np.sort(-a, axis=1)
    aL = srt[:, L - 1:L]
    return np.abs(a - aL) <= rel * np.abs(aL)


# ---------------------------------------------------------------------------
# a-3: set sketches  (Def 8 P:657 + Alg 3; Def 10 P:729-732 + Alg 5)
# ---------------------------------------------------------------------------


def _check_offsets(offsets: np.ndarray) -> np.ndarray:
    o = np.asarray(offsets, dtype=np.int64)
    if o.ndim != 1 or o.size < 2 or o[0] != 0 or np.any(np.diff(o) <= 0):
        raise ValueError("set offsets must start at 0 and be strictly increasing (Def 2: m >= 1)")
    return o


def sketch_binary(codes: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """Binary Bloom filter / set sketch B = OR_{v in V} H(v) (Def 10 P:731,
    Alg 5 lines 3-5; S = B, Alg 5 line 5).  Returns uint32 ``[n][m/32]``."""
    o = _check_offsets(offsets)
    return np.bitwise_or.reduceat(np.asarray(codes, dtype=np.uint32), o[:-1], axis=0)


def sketch_count(codes: np.ndarray, offsets: np.ndarray, m: int) -> np.ndarray:
    """Count Bloom filter c_i = sum_j H(v_j)_i (Def 8, Alg 3 line 4).
    Reading R14: stored as uint8, saturating at 255.  Returns uint8 ``[n][m]``."""
    o = _check_offsets(offsets)
    bits = unpack_bits(codes, m).astype(np.int64)
    c = np.add.reduceat(bits, o[:-1], axis=0)
    return np.minimum(c, 255).astype(np.uint8)


# ---------------------------------------------------------------------------
# a-5: filter scores  (Alg 6 line 12 P:797; readings R1, R2)
# ---------------------------------------------------------------------------


def popcount_rows(words: np.ndarray) -> np.ndarray:
    """Number of set bits per row of a uint32 word array (int64 ``[n]``)."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    return np.bitwise_count(w).astype(np.int64).sum(axis=1)


def hamming_scores(SQ: np.ndarray, S: np.ndarray) -> np.ndarray:
    """Hamming(S_Q, S^(i)) = popcount(S_Q XOR S^(i)) for every DB sketch
    (Alg 6 line 12 P:797; "XOR and popcount" P:725).  SQ: uint32 ``[m/32]``,
    S: uint32 ``[n][m/32]``.  Returns int64 ``[n]``."""
    x = np.bitwise_xor(np.asarray(S, dtype=np.uint32), np.asarray(SQ, dtype=np.uint32)[None, :])
    return popcount_rows(x)


def count_l2_scores(CQ: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Reading R2 (count-Bloom score): squared L2 distance between counter
    vectors, sum_j (C_Q[j] - C_i[j])^2, exact int64.  Returns int64 ``[n]``."""
    diff = np.asarray(C, dtype=np.int64) - np.asarray(CQ, dtype=np.int64)[None, :]
    return (diff * diff).sum(axis=1)


def overlap_scores(SQ: np.ndarray, S: np.ndarray, kind: str = "binary") -> np.ndarray:
    """The OVERLAP filter score (reading R24, SURVEY A1 flag): the shared-bit
    count popc(S_Q AND S^(i)) the north_star's scan computes ("ANDs and
    popcounts"), or for count sketches the counter dot product
    sum_j C_Q[j] C_i[j] (Theorem 2's collision count).  Higher is
    closer; returns int64 ``[n]``."""
    if kind == "binary":
        a = np.bitwise_and(np.asarray(S, dtype=np.uint32), np.asarray(SQ, dtype=np.uint32)[None, :])
        return popcount_rows(a)
    C = np.asarray(S, dtype=np.int64)
    return (C * np.asarray(SQ, dtype=np.int64)[None, :]).sum(axis=1)


def count_l1_scores(CQ: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Reading R26 (SURVEY A2's L1 flag): L1 distance between counter vectors,
    sum_j |C_Q[j] - C_i[j]|, exact int64.  Returns int64 ``[n]``."""
    diff = np.asarray(C, dtype=np.int64) - np.asarray(CQ, dtype=np.int64)[None, :]
    return np.abs(diff).sum(axis=1)


# ---------------------------------------------------------------------------
# a-6: top-T candidate selection  (Alg 6 lines 10-18 P:795-806; readings R3, R4)
# ---------------------------------------------------------------------------


def select_top_T(scores: np.ndarray, T: int) -> np.ndarray:
    """F2 = the T sets with smallest filter score (Alg 6 lines 10-18: a
    T-capacity max-heap keeps the T closest).  Readings R3/R4: one budget T,
    ties broken by ascending set id, exactly min(T, n) ids.  Returned in
    (score, id) order, int64."""
    sc = np.asarray(scores)
    ids = np.arange(sc.shape[0], dtype=np.int64)
    order = np.lexsort((ids, sc))
    return order[:min(T, sc.shape[0])].astype(np.int64)


# ---------------------------------------------------------------------------
# BioVSS++ stage 1: the inverted-index gate  (Alg 6 lines 1, 3-9 P:779-792;
# Def 9 / Alg 4; defaults A = 3, M = 1 P:968; reading R27)
# ---------------------------------------------------------------------------


def stage1_positions(CQ: np.ndarray, A: int) -> np.ndarray:
    """P = {pi(i) : i in [1, A]} with pi = ArgsortDescending(C_Q) (Alg 6 lines
    3-4): the A positions of the query's count Bloom filter with the
    largest counts.  Reading R27: among equal counts the lower position comes
    first (a stable descending sort).  Returns int64 ``[min(A, m)]``."""
    CQ = np.asarray(CQ, dtype=np.int64)
    order = np.argsort(-CQ, kind="stable")
    return order[:min(int(A), CQ.shape[0])].astype(np.int64)


def inverted_index(C: np.ndarray) -> list:
    """Build_Inverted_Index (Alg 4; Def 9): for every position i a
    list of (j, c_i^(j)) over ALL sets j (zero counts included, Alg 4 lines
    3-6), sorted by descending count (line 8; ties keep ascending j)."""
    C = np.asarray(C, dtype=np.int64)
    n, m = C.shape
    I = []
    for i in range(m):
        lst = [(j, int(C[j, i])) for j in range(n)]
        lst.sort(key=lambda t: -t[1])  # Python's sort is stable: equal counts keep ascending j
        I.append(lst)
    return I


def stage1_gate_loops(I: list, P, M: int) -> np.ndarray:
    """F1 of Alg 6 lines 5-9 written as its loops over the inverted
    lists: for p in P, for (i, c) in I[p]: if c >= M, add i.  Returns the sorted
    ids (int64).  Slow; used on small inputs only."""
    F1 = set()
    for p in P:
        for i, c in I[int(p)]:
            if c >= M:
                F1.add(i)
    return np.array(sorted(F1), dtype=np.int64)


def stage1_gate(C: np.ndarray, P, M: int) -> np.ndarray:
    """F1 as a mask over the count Bloom filters C [n][m]: set i passes iff
    C_i[p] >= M for some p in P (the same set as stage1_gate_loops).  For a
    binary index the counts are the binary sketch bits (S = (C > 0), Def 8 /
    Def 10), which decides the gate exactly for M <= 1.  Returns bool ``[n]``."""
    C = np.asarray(C, dtype=np.int64)
    P = np.asarray(P, dtype=np.int64)
    if P.size == 0:
        return np.zeros(C.shape[0], dtype=bool) if M > 0 else np.ones(C.shape[0], dtype=bool)
    return (C[:, P] >= M).any(axis=1)


# ---------------------------------------------------------------------------
# BioVSS Alg 2: Hamming-Hausdorff candidate scan over per-vector codes
# (Haus^H P:378, described P:396)
# ---------------------------------------------------------------------------


def hamming_matrix(QH: np.ndarray, VH: np.ndarray) -> np.ndarray:
    """hamming(q, v) = popcount(h_q XOR h_v) for every pair of packed codes
    (uint32 rows), int64 ``[|Q|][|V|]``."""
    QH = np.asarray(QH, dtype=np.uint32)
    VH = np.asarray(VH, dtype=np.uint32)
    x = np.bitwise_xor(QH[:, None, :], VH[None, :, :])
    return np.bitwise_count(x).astype(np.int64).sum(axis=2)


def haus_hamming(QH: np.ndarray, VH: np.ndarray) -> int:
    """Haus^H(Q^H, H_j) (Alg 2 line 7): Def 4's aggregation with
    hamming(q, v) in place of dist:
    max( max_q min_v ham, max_v min_q ham )."""
    Hm = hamming_matrix(QH, VH)
    return int(max(Hm.min(axis=1).max(), Hm.min(axis=0).max()))


def alg2_candidates(QH: np.ndarray, codes: np.ndarray, offsets: np.ndarray, c: int):
    """Alg 2 lines 6-9: d_H for every database set, then F = the c
    sets with the smallest d_H (readings R3/R4: exactly min(c, n), ties by
    ascending id).  Returns (ids in (d_H, id) order, d_H of every set)."""
    o = _check_offsets(offsets)
    n = o.shape[0] - 1
    dH = np.array([haus_hamming(QH, codes[o[j]:o[j + 1]]) for j in range(n)], dtype=np.int64)
    return select_top_T(dH, c), dH


# ---------------------------------------------------------------------------
# a-7: Hausdorff distance  (Def 4)
# ---------------------------------------------------------------------------


def pairwise_dist(Q: np.ndarray, V: np.ndarray) -> np.ndarray:
    """dist(q, v) = ||q - v||_2 for all pairs (Def 4), by direct
    differences in fp64.  Returns ``[|Q|][|V|]``."""
    Q = np.asarray(Q, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    diff = Q[:, None, :] - V[None, :, :]
    return np.sqrt((diff * diff).sum(axis=2))


def hausdorff_from_dist(Dm: np.ndarray) -> float:
    """The aggregation of Def 4 on a distance matrix Dm[q][v]:
    max( max_q min_v Dm, max_v min_q Dm )  (Example 2: directed values
    then the final max)."""
    Dm = np.asarray(Dm, dtype=np.float64)
    return float(max(Dm.min(axis=1).max(), Dm.min(axis=0).max()))


def hausdorff(Q: np.ndarray, V: np.ndarray) -> float:
    """Haus(Q, V) of Def 4, fp64 direct differences (reading R9)."""
    return hausdorff_from_dist(pairwise_dist(Q, V))


def meanmin_from_dist(Dm: np.ndarray) -> float:
    """MeanMin distance d_mean-min(A, B) = 1/|A| sum_{a in A} min_b d(a, b)
    (P:196), on Dm[a][b]."""
    Dm = np.asarray(Dm, dtype=np.float64)
    return float(Dm.min(axis=1).mean())


def min_from_dist(Dm: np.ndarray) -> float:
    """Min distance d_min(A, B) = min_{a,b} d(a, b)."""
    return float(np.min(Dm))


METRICS = ("hausdorff", "meanmin", "min")


def set_distance(Q: np.ndarray, V: np.ndarray, metric: str = "hausdorff") -> float:
    """The rerank distance between the query set Q and a database set V, fp64
    direct differences: Hausdorff (Def 4; the paper's metric), or
    the §3.2 alternatives: MeanMin d_mean-min(Q, V)
    (A = the query set, reading R23) and Min d_min(Q, V)."""
    Dm = pairwise_dist(Q, V)
    if metric == "hausdorff":
        return hausdorff_from_dist(Dm)
    if metric == "meanmin":
        return meanmin_from_dist(Dm)
    if metric == "min":
        return min_from_dist(Dm)
    raise ValueError(metric)


def hausdorff_gram(Q: np.ndarray, V: np.ndarray) -> float:
    """Hausdorff through the fp64 Gram form ||q||^2 + ||v||^2 - 2 q.v (BLAS),
    clamped at 0 before sqrt.  Used for brute force at scale; agrees with
    ``hausdorff`` to ~1e-7 absolute (self-test in tests)."""
    Q = np.asarray(Q, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    d2 = (Q * Q).sum(1)[:, None] + (V * V).sum(1)[None, :] - 2.0 * (Q @ V.T)
    return hausdorff_from_dist(np.sqrt(np.maximum(d2, 0.0)))


def refine(Q: np.ndarray, cand: np.ndarray, vectors: np.ndarray, offsets: np.ndarray,
           metric: str = "hausdorff") -> np.ndarray:
    """Alg 6 lines 19-22 (iterating F2 per reading R5): exact
    Haus(Q, V_i) (or the MeanMin / Min alternative, ``set_distance``) for every
    candidate i.  Returns fp64 ``[len(cand)]``."""
    o = np.asarray(offsets, dtype=np.int64)
    out = np.empty(len(cand), dtype=np.float64)
    for t, i in enumerate(np.asarray(cand, dtype=np.int64)):
        out[t] = set_distance(Q, vectors[o[i]:o[i + 1]], metric)
    return out


# ---------------------------------------------------------------------------
# a-8: final top-k  (Alg 6 line 23 P:814; Def 5; reading R4, R16)
# ---------------------------------------------------------------------------


def top_k(ids: np.ndarray, dist: np.ndarray, k: int):
    """R = the k candidates with the smallest Haus (Alg 6 line 23),
    sorted by (distance, id); fewer than k candidates pad with (-1, +inf)."""
    ids = np.asarray(ids, dtype=np.int64)
    dist = np.asarray(dist, dtype=np.float64)
    order = np.lexsort((ids, dist))[:k]
    out_ids = np.full(k, -1, dtype=np.int64)
    out_d = np.full(k, np.inf, dtype=np.float64)
    out_ids[:len(order)] = ids[order]
    out_d[:len(order)] = dist[order]
    return out_ids, out_d


# ---------------------------------------------------------------------------
# The whole path: Alg 6 with stage 1 open (reading R6), and brute force
# ---------------------------------------------------------------------------


class OracleIndex:
    """Index state of Algs 1, 3, 5 for one database (P:323-343, P:665-682,
    P:738-757): W, per-vector codes D^H, per-set sketches."""

    def __init__(self, vectors, offsets, m, s, L, seed, sketch="binary", W=None, score="default", sketches=None):
        """``sketches``: database sketches handed in from the stage under test
        (stage-wise parity: each stage is fed the previous stage's
        output), skipping the database encode; queries are still encoded here."""
        self.vectors = np.ascontiguousarray(vectors, dtype=np.float32)
        self.offsets = _check_offsets(offsets)
        if self.offsets[-1] != self.vectors.shape[0]:
            raise ValueError("offsets[-1] must equal the number of vectors")
        self.d = self.vectors.shape[1]
        self.m, self.s, self.L, self.seed = m, s, L, seed
        self.kind = sketch
        self.score = score  # "default" (Hamming / L2^2), "overlap" (descending, R24), "binarized" (R25)
        self.W = projection(seed, m, s, self.d) if W is None else np.asarray(W, dtype=np.uint16)
        if sketches is not None:
            self.codes = None
            self.sketches = np.asarray(sketches)
            if self.sketches.shape[0] != self.n or sketch not in ("binary", "count"):
                raise ValueError("sketches must hold one row per set")
            return
        self.codes = encode(self.vectors, self.W, L)
        if sketch == "binary":
            self.sketches = sketch_binary(self.codes, self.offsets)
        elif sketch == "count":
            self.sketches = sketch_count(self.codes, self.offsets, m)
        else:
            raise ValueError(sketch)

    @property
    def n(self) -> int:
        return self.offsets.shape[0] - 1

    def query_sketch(self, Q):
        """Alg 6 lines 1-2: encode the query set and fold it."""
        codes = encode(np.asarray(Q, dtype=np.float32), self.W, self.L)
        off = np.array([0, codes.shape[0]], dtype=np.int64)
        if self.kind == "binary":
            return sketch_binary(codes, off)[0]
        return sketch_count(codes, off, self.m)[0]

    def scores(self, Q) -> np.ndarray:
        """Filter scores, smaller = closer (the order select_top_T ranks by)."""
        sq = self.query_sketch(Q)
        if self.score == "overlap":
            return -overlap_scores(sq, self.sketches, self.kind)
        if self.score == "l1" and self.kind == "count":  # R26
            return count_l1_scores(sq, self.sketches)
        if self.score == "binarized" and self.kind == "count":  # R25: Hamming between (C_Q > 0), (C_i > 0)
            return hamming_scores(pack_bits(sq[None, :] > 0)[0], pack_bits(self.sketches > 0))
        if self.kind == "binary":
            return hamming_scores(sq, self.sketches)
        return count_l2_scores(sq, self.sketches)

    def filter(self, Q, T: int) -> np.ndarray:
        return select_top_T(self.scores(Q), T)

    def query_counts(self, Q) -> np.ndarray:
        """C_Q = Gen_Count_Bloom_Filter(Q) (Alg 6 line 1 P:779; Alg 3 / Def 8)."""
        codes = encode(np.asarray(Q, dtype=np.float32), self.W, self.L)
        return sketch_count(codes, np.array([0, codes.shape[0]], dtype=np.int64), self.m)[0]

    def db_counts(self) -> np.ndarray:
        """The database counters the gate reads: count sketches as stored, or the binary sketch bits (0/1),
        which decide C_i[p] >= M exactly for M <= 1 (S = (C > 0))."""
        if self.kind == "count":
            return np.asarray(self.sketches, dtype=np.int64)
        return unpack_bits(self.sketches, self.m).astype(np.int64)

    def filter_gated(self, Q, T: int, A: int, M: int) -> np.ndarray:
        """Alg 6 lines 1-18: F1 by the inverted-index gate (top-A query positions, count >= M),
        then F2 = the first T of F1 by (score, id); |F1| < T gives F2 = F1."""
        P = stage1_positions(self.query_counts(Q), A)
        gate = stage1_gate(self.db_counts(), P, M)
        sc = self.scores(Q)
        ids = np.flatnonzero(gate)
        order = np.lexsort((ids, sc[ids]))
        return ids[order][:min(T, ids.shape[0])].astype(np.int64)

    def search_gated(self, Q, k: int, T: int, A: int, M: int):
        """BioVSS++ (Alg 6) with stage 1 enabled: gate, sketch filter, exact Hausdorff rerank, top-k."""
        if T < k:
            raise ValueError("T < k (reading R16)")
        cand = self.filter_gated(Q, T, A, M)
        return top_k(cand, refine(Q, cand, self.vectors, self.offsets), k)

    def search_alg2(self, Q, k: int, c: int):
        """BioVSS (Alg 2): Haus^H over the per-vector codes to c candidates, exact Hausdorff
        rerank (lines 10-13), top-k (line 14).  Needs the database codes (built unless sketches were given)."""
        if self.codes is None:
            raise ValueError("Alg 2 needs the database codes")
        QH = encode(np.asarray(Q, dtype=np.float32), self.W, self.L)
        cand, _ = alg2_candidates(QH, self.codes, self.offsets, c)
        return top_k(cand, refine(Q, cand, self.vectors, self.offsets), k)

    def set_vectors(self, i: int) -> np.ndarray:
        return self.vectors[self.offsets[i]:self.offsets[i + 1]]

    def search(self, Q, k: int, T: int, metric: str = "hausdorff"):
        """Alg 6 with F1 = D: filter to T candidates, exact
        Hausdorff (or MeanMin / Min) rerank, top-k by (distance, id)."""
        if T < k:
            raise ValueError("T < k (reading R16)")
        cand = self.filter(Q, T)
        dist = refine(Q, cand, self.vectors, self.offsets, metric)
        return top_k(cand, dist, k)

    def bruteforce(self, Q, k: int, limit: int | None = None, metric: str = "hausdorff"):
        """Exact top-k over all sets ("precise calculations according to
        Definition 4")."""
        n = self.n if limit is None else min(limit, self.n)
        ids = np.arange(n, dtype=np.int64)
        dist = refine(Q, ids, self.vectors, self.offsets, metric)
        return top_k(ids, dist, k)


def bruteforce_topk(Q, vectors, offsets, k: int, ids=None):
    """Exact top-k Hausdorff over the given set ids (all sets by default)."""
    o = np.asarray(offsets, dtype=np.int64)
    if ids is None:
        ids = np.arange(o.shape[0] - 1, dtype=np.int64)
    dist = refine(Q, ids, vectors, o)
    return top_k(ids, dist, k)


def recall_at_k(R: np.ndarray, G: np.ndarray) -> float:
    """Recall@k = |R_k(Q) ∩ G_k(Q)| / |G_k(Q)|."""
    g = set(int(x) for x in G if x >= 0)
    r = set(int(x) for x in R if x >= 0)
    return len(r & g) / max(1, len(g))
