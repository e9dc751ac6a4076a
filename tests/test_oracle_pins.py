"""Pins for the CPU oracle (-m "not gpu").

Each test ties an oracle function to something other than itself: a value the
paper prints (tests/golden/, cited), a closed form, a published known answer,
an invariant the paper states, or a brute-force / independent formulation on
tiny inputs.  Chosen so that a dropped term, a wrong sign or index, or a
transposed operand in the oracle fails at least one of them.
"""
import json
import os

import numpy as np
import pytest

from oracle import bvss_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------- projection W

def test_splitmix64_known_answer():
    g = gold("splitmix64.json")
    it = O.splitmix64_stream(g["state"])
    assert [next(it) for _ in range(8)] == [int(h, 16) for h in g["outputs_hex"]]


def test_projection_row0_from_published_draws():
    """Row 0 seeds its SplitMix64 state with seed ^ (0 * C) = seed, so at seed 0
    its draws are the published state-0 outputs (tests/golden/splitmix64.json).
    d = 64: 2^64 mod 64 = 0, no rejection, dims = u mod 64 = the low 6 bits:
    0xaf & 63 = 47, 0xf4 & 63 = 52, 0x4f & 63 = 15, 0xec & 63 = 44,
    0x9b & 63 = 27, 0xea & 63 = 42 (all distinct) -> sorted [15 27 42 44 47 52]
    (BJ cfg1 shape: s = 6 ones per row, d = 64; reading R7)."""
    W = O.projection(0, 4, 6, 64)
    assert W[0].tolist() == [15, 27, 42, 44, 47, 52]
    # d = 384 (not a power of two; 2^64 mod 384 = 256 != 0, but no published draw lies in the
    # rejected tail [2^64 - 256, 2^64)): dims = u mod 384 of the first 8 draws, first 8 distinct kept
    g = gold("splitmix64.json")
    draws = [int(h, 16) for h in g["outputs_hex"]]
    assert (1 << 64) % 384 == 256 and all(u < (1 << 64) - 256 for u in draws)
    want = []
    for u in draws:
        if u % 384 not in want:
            want.append(u % 384)
    assert len(want) == 8
    assert O.projection(0, 2, 8, 384)[0].tolist() == sorted(want)
    # row 1 does NOT reuse the state-0 stream (per-row seed mixing seed ^ (j * 0xD1B54A32D192ED03))
    assert O.projection(0, 2, 6, 64)[1].tolist() != [15, 27, 42, 44, 47, 52]


@pytest.mark.parametrize("m,s,d", [(512, 6, 64), (64, 8, 384), (32, 12, 768), (40, 3, 3)])
def test_projection_rows_are_s_distinct_sorted_dims(m, s, d):
    W = O.projection(7, m, s, d)
    assert W.shape == (m, s) and W.dtype == np.uint16
    assert np.all(W < d)
    assert np.all(np.diff(W.astype(np.int64), axis=1) > 0)  # sorted, hence distinct
    assert np.array_equal(W, O.projection(7, m, s, d))      # deterministic
    assert not np.array_equal(W, O.projection(8, m, s, d)) or s == d


def test_projection_uniform_over_dims():
    # "uniformly sampled input dims" (BJ cfg1): column usage ~ uniform (chi-square)
    m, s, d = 4096, 6, 64
    W = O.projection(3, m, s, d)
    counts = np.bincount(W.ravel(), minlength=d)
    exp = m * s / d
    chi2 = ((counts - exp) ** 2 / exp).sum()
    assert chi2 < 140.0  # dof 63: p ~ 1e-7 threshold
    # rows are not all identical and all C(d,s) patterns are possible in principle
    assert len({tuple(r) for r in W.tolist()}) > m - 5


# ----------------------------------------------------------------- near-tie rows

def test_near_tie_rows_hand_built():
    """The code-parity exemption (BJ north_star: rows whose activation is within
    1e-5 relative of the L-th largest).  Hand-built activations, identity-like W
    (s = 3 dims per row, the unused dims are exact zeros):
      row 0: x0 + x1 + x2 = 1e4 + 1e-3 - 1e4 -> fp64 1e-3, but fp32 left to right 9.765625e-4
      row 1: x1 = 1e-3 exactly (the L-th largest for L = 2)
      row 2: 5.0 (largest), row 3: -5.0, row 4: 0.0
      rows 5/6: 1e-3 (1 - 0.5e-5) (inside the band) / 1e-3 (1 - 2e-5) (outside)
    Pins: the band is rel * |a_(L)| with rel = 1e-5; a_(L) is the L-th (not the
    (L+1)-th or (L-1)-th) largest; the activation is taken in fp64 (in fp32 row 0
    would sit 2.3 % below a_(L) and not be flagged)."""
    x = np.zeros(12)
    x[0], x[1], x[2] = 1e4, 1e-3, -1e4
    x[5], x[6] = 5.0, -5.0
    x[8] = 1e-3 * (1 - 0.5e-5)
    x[9] = 1e-3 * (1 - 2e-5)
    W = np.array([[0, 1, 2], [1, 3, 4], [3, 4, 5], [3, 4, 6], [3, 4, 7], [3, 4, 8], [3, 4, 9]], dtype=np.uint16)
    a32 = O.activations(x[None, :].astype(np.float32), W)[0]
    assert a32[0] == np.float32(9.765625e-4)  # the fp32 order really loses the 1e-3 (precondition)
    got = O.near_tie_rows(x[None, :], W, 2)[0]
    assert got.tolist() == [True, True, False, False, False, True, False]
    # L = 1: a_(1) = 5.0 -> only row 2
    assert O.near_tie_rows(x[None, :], W, 1)[0].tolist() == [False, False, True, False, False, False, False]
    # a wider band (rel = 3e-5) also takes row 6
    assert O.near_tie_rows(x[None, :], W, 2, rel=3e-5)[0].tolist() == [True, True, False, False, False, True, True]


# ----------------------------------------------------------------- activations

def test_activations_decode_projection_structure():
    # v_i = 2^i (exact in fp32): (W v)_j = sum_{i in S_j} 2^i, whose binary
    # digits are exactly row j's index set -> any wrong index, dropped or
    # duplicated term is visible.
    d, m, s = 20, 50, 5
    W = O.projection(11, m, s, d)
    v = (2.0 ** np.arange(d)).astype(np.float32)[None, :]
    a = O.activations(v, W)[0].astype(np.int64)
    for j in range(m):
        bits = [i for i in range(d) if (a[j] >> i) & 1]
        assert bits == sorted(W[j].tolist())


def test_activations_identity_and_fp64_bound():
    rng = np.random.default_rng(0)
    d = 16
    W = np.arange(d, dtype=np.uint16)[:, None]  # identity, s = 1
    V = rng.standard_normal((5, d)).astype(np.float32)
    assert np.array_equal(O.activations(V, W), V)
    # fp32 left-to-right sum of s terms is within s * 2^-24 * sum|v| of the exact sum
    W = O.projection(5, 256, 12, 384)
    V = rng.standard_normal((64, 384)).astype(np.float32)
    a32 = O.activations(V, W).astype(np.float64)
    a64 = O.activations_fp64(V, W)
    absum = np.zeros_like(a64)
    for t in range(W.shape[1]):
        absum += np.abs(V[:, W[:, t]].astype(np.float64))
    assert np.all(np.abs(a32 - a64) <= 12 * 2.0 ** -24 * absum + 1e-30)


def test_activations_left_to_right_order():
    # reading R8: ((0 + v0) + v1) + v2 in fp32; a different association differs here
    W = np.array([[0, 1, 2]], dtype=np.uint16)
    v = np.array([[1.0, 2.0 ** -24, 2.0 ** -24]], dtype=np.float32)
    assert O.activations(v, W)[0, 0] == np.float32(1.0)                 # (1+e)+e rounds to 1 twice
    assert np.float32(1.0) + (np.float32(2.0 ** -24) + np.float32(2.0 ** -24)) != np.float32(1.0)


# ----------------------------------------------------------------- WTA

def test_wta_paper_example():
    g = gold("wta_identity.json")
    a = np.array([g["v"]], dtype=np.float32)
    h = O.wta(a, g["L"])
    assert np.flatnonzero(h[0]).tolist() == g["bits"]


def test_wta_L_equals_m_all_ones_and_exactly_L():
    rng = np.random.default_rng(1)
    a = rng.standard_normal((100, 64)).astype(np.float32)
    assert O.wta(a, 64).all()
    for L in (1, 5, 16, 63):
        h = O.wta(a, L)
        assert np.all(h.sum(1) == L)
        # definition: every winner >= every loser
        for r in range(a.shape[0]):
            assert a[r][h[r]].min() >= a[r][~h[r]].max()


def test_wta_ties_go_to_lower_index():
    a = np.array([[1.0, 3.0, 3.0, 3.0, 0.0, 3.0]], dtype=np.float32)
    assert np.flatnonzero(O.wta(a, 2)[0]).tolist() == [1, 2]
    assert np.flatnonzero(O.wta(a, 5)[0]).tolist() == [0, 1, 2, 3, 5]
    z = np.array([[0.0, -0.0, -0.0, 0.0]], dtype=np.float32)  # -0 == +0: pure index order
    assert np.flatnonzero(O.wta(z, 2)[0]).tolist() == [0, 1]


def test_wta_matches_full_sort_and_is_permutation_equivariant():
    rng = np.random.default_rng(2)
    a = rng.standard_normal((50, 128)).astype(np.float32)
    h = O.wta(a, 20)
    for r in range(50):
        ranked = sorted(range(128), key=lambda j: (-float(a[r, j]), j))[:20]
        assert sorted(ranked) == np.flatnonzero(h[r]).tolist()
    perm = rng.permutation(128)
    assert np.array_equal(O.wta(a[:, perm], 20), h[:, perm])


def test_pack_bits_layout():
    h = np.zeros((1, 64), dtype=bool)
    h[0, 33] = True
    h[0, 0] = True
    w = O.pack_bits(h)
    assert w.tolist() == [[1, 2]]
    assert np.array_equal(O.unpack_bits(w, 64), h)


def test_encode_codes_have_exactly_L_ones():
    rng = np.random.default_rng(3)
    V = rng.standard_normal((300, 64)).astype(np.float32)
    W = O.projection(0, 512, 6, 64)
    codes = O.encode(V, W, 16)
    assert codes.shape == (300, 16)
    assert np.all(O.popcount_rows(codes) == 16)


# ----------------------------------------------------------------- sketches

def _codes_from_bits(lists, m):
    h = np.zeros((len(lists), m), dtype=bool)
    for r, bits in enumerate(lists):
        h[r, bits] = True
    return O.pack_bits(h)


def test_sketch_single_vector_equals_code_and_counts():
    rng = np.random.default_rng(4)
    V = rng.standard_normal((10, 32)).astype(np.float32)
    W = O.projection(1, 256, 4, 32)
    codes = O.encode(V, W, 8)
    off = np.arange(11, dtype=np.int64)
    assert np.array_equal(O.sketch_binary(codes, off), codes)
    C = O.sketch_count(codes, off, 256)
    assert np.array_equal(C.astype(bool), O.unpack_bits(codes, 256))


def test_sketch_disjoint_codes_and_counting_identities():
    m = 128
    codes = _codes_from_bits([[0, 1, 2], [10, 11, 12], [100, 101, 127], [0, 11, 127]], m)
    off = np.array([0, 3, 4], dtype=np.int64)
    S = O.sketch_binary(codes, off)
    C = O.sketch_count(codes, off, m)
    assert O.popcount_rows(S).tolist() == [9, 3]            # disjoint -> |V| * L
    assert C.astype(np.int64).sum(1).tolist() == [9, 3]     # sum C = |V| * L
    assert np.array_equal(O.unpack_bits(S, m), C > 0)      # S = (C > 0)
    assert C[0, 0] == 1 and C[1, 0] == 1 and C[1, 127] == 1


def test_sketch_bounds_and_saturation():
    rng = np.random.default_rng(5)
    V = rng.standard_normal((400, 48)).astype(np.float32)
    W = O.projection(2, 512, 6, 48)
    L = 16
    codes = O.encode(V, W, L)
    sizes = rng.integers(1, 20, 40)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    codes = codes[:off[-1]]
    p = O.popcount_rows(O.sketch_binary(codes, off))
    assert np.all(p >= L) and np.all(p <= np.minimum(512, sizes * L))
    C = O.sketch_count(codes, off, 512)
    assert np.array_equal(C.astype(np.int64).sum(1), sizes * L)
    same = np.repeat(codes[:1], 300, axis=0)               # 300 identical codes
    Cs = O.sketch_count(same, np.array([0, 300]), 512)
    assert Cs.max() == 255 and np.all(Cs[O.unpack_bits(codes[:1], 512)] == 255)


# ----------------------------------------------------------------- scores

def test_hamming_matches_bit_loop_and_identities():
    rng = np.random.default_rng(6)
    m = 96
    S = rng.integers(0, 2 ** 32, (20, m // 32), dtype=np.uint64).astype(np.uint32)
    q = S[3]
    ham = O.hamming_scores(q, S)
    bq = O.unpack_bits(q[None], m)[0]
    for i in range(20):
        bi = O.unpack_bits(S[i:i + 1], m)[0]
        assert ham[i] == sum(int(bq[j] != bi[j]) for j in range(m))
    assert ham[3] == 0
    comp = np.bitwise_not(q)
    assert O.hamming_scores(comp, q[None])[0] == m
    pa = O.popcount_rows(S)
    pq = O.popcount_rows(q[None])[0]
    pand = O.popcount_rows(np.bitwise_and(S, q[None]))
    assert np.array_equal(ham, pq + pa - 2 * pand)          # reading R1
    assert all(O.hamming_scores(S[i], S[j:j + 1])[0] == O.hamming_scores(S[j], S[i:i + 1])[0]
               for i in range(5) for j in range(5))


def test_count_l2_reduces_to_hamming_on_binary_counters():
    rng = np.random.default_rng(7)
    m = 64
    S = rng.integers(0, 2 ** 32, (10, 2), dtype=np.uint64).astype(np.uint32)
    C = O.unpack_bits(S, m).astype(np.uint8)
    for i in range(10):
        assert np.array_equal(O.count_l2_scores(C[i], C), O.hamming_scores(S[i], S))
    C2 = np.array([[3, 0, 1]], dtype=np.uint8)
    assert O.count_l2_scores(np.array([1, 2, 1], np.uint8), C2)[0] == 4 + 4 + 0


# ----------------------------------------------------------------- top-T

def test_overlap_scores_bit_loop_and_identities():
    """OVERLAP (R24): popc(S_Q AND S_i) by a per-bit Python loop; Hamming =
    p_Q + p_i - 2 overlap against the independent XOR form; count sketches:
    the dot product by a loop and L2^2 = |C_Q|^2 + |C_i|^2 - 2 dot; the
    ranking is by descending overlap, ties by id."""
    rng = np.random.default_rng(21)
    m = 96
    S = rng.integers(0, 2**32, size=(40, m // 32), dtype=np.uint64).astype(np.uint32)
    SQ = rng.integers(0, 2**32, size=(m // 32,), dtype=np.uint64).astype(np.uint32)
    ov = O.overlap_scores(SQ, S)
    for i in range(S.shape[0]):
        loop = sum(((int(S[i, w]) >> b) & (int(SQ[w]) >> b) & 1) for w in range(m // 32) for b in range(32))
        assert ov[i] == loop
    pq = O.popcount_rows(SQ[None, :])[0]
    assert np.array_equal(O.hamming_scores(SQ, S), pq + O.popcount_rows(S) - 2 * ov)
    C = rng.integers(0, 6, size=(30, 20)).astype(np.uint8)
    CQ = rng.integers(0, 6, size=(20,)).astype(np.uint8)
    dot = O.overlap_scores(CQ, C, "count")
    for i in range(C.shape[0]):
        assert dot[i] == sum(int(C[i, j]) * int(CQ[j]) for j in range(20))
    n2 = lambda x: (x.astype(np.int64) ** 2).sum(-1)
    assert np.array_equal(O.count_l2_scores(CQ, C), n2(CQ) + n2(C) - 2 * dot)
    # descending overlap, ties by id: a set equal to the query's sketch and a superset come first
    S2 = np.array([[0x0F], [0xFF], [0x0F], [0x01]], dtype=np.uint32)
    assert O.select_top_T(-O.overlap_scores(np.array([0x0F], dtype=np.uint32), S2), 4).tolist() == [0, 1, 2, 3]


def test_binarized_count_score_equals_binary_sketch_hamming():
    """BINARIZED (R25): Hamming between the binarised count sketches equals the
    Hamming of the OR-fold binary sketches of the same codes (Def 8 vs Def 10:
    S = (C > 0)), for every query, through two different oracle paths."""
    rng = np.random.default_rng(4)
    sizes = rng.integers(1, 7, size=60)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    V = rng.normal(size=(off[-1], 24)).astype(np.float32)
    cnt = O.OracleIndex(V, off, 64, 3, 5, 9, sketch="count", score="binarized")
    bin_ = O.OracleIndex(V, off, 64, 3, 5, 9, sketch="binary")
    for q in range(4):
        Q = rng.normal(size=(int(rng.integers(1, 5)), 24)).astype(np.float32)
        assert np.array_equal(cnt.scores(Q), bin_.scores(Q))
        assert np.array_equal(cnt.filter(Q, 10), bin_.filter(Q, 10))


def test_count_l1_scores_loop_and_binary_reduction():
    """L1 (R26): a per-counter loop; on 0/1 counters L1 = L2^2 = Hamming."""
    rng = np.random.default_rng(5)
    C = rng.integers(0, 255, size=(25, 16)).astype(np.uint8)
    CQ = rng.integers(0, 255, size=(16,)).astype(np.uint8)
    l1 = O.count_l1_scores(CQ, C)
    for i in range(C.shape[0]):
        assert l1[i] == sum(abs(int(C[i, j]) - int(CQ[j])) for j in range(16))
    B01 = rng.integers(0, 2, size=(25, 64)).astype(np.uint8)
    BQ = rng.integers(0, 2, size=(64,)).astype(np.uint8)
    ham = O.hamming_scores(O.pack_bits(BQ[None, :] > 0)[0], O.pack_bits(B01 > 0))
    assert np.array_equal(O.count_l1_scores(BQ, B01), ham)
    assert np.array_equal(O.count_l2_scores(BQ, B01), ham)


def test_select_top_T_ties_by_id_and_nesting():
    sc = np.array([5, 1, 3, 1, 3, 3, 0, 9], dtype=np.int64)
    assert O.select_top_T(sc, 4).tolist() == [6, 1, 3, 2]
    assert sorted(O.select_top_T(sc, 100).tolist()) == list(range(8))
    rng = np.random.default_rng(8)
    sc = rng.integers(0, 20, 500)
    full = sorted(range(500), key=lambda i: (sc[i], i))
    for T in (1, 10, 77, 499, 500):
        got = O.select_top_T(sc, T)
        assert got.tolist() == full[:T]
        assert set(O.select_top_T(sc, max(1, T // 2)).tolist()) <= set(got.tolist())


# ----------------------------------------------------------------- Hausdorff

def test_hausdorff_section32_matrices():
    g = gold("hausdorff_section32.json")
    for c in g["cases"]:
        M = np.array(c["matrix"], dtype=np.float64)       # rows = target, cols = Q
        DqT = M.T                                          # rows = Q
        if "hausdorff" in c:
            assert O.hausdorff_from_dist(DqT) == c["hausdorff"]
            assert O.hausdorff_from_dist(M) == c["hausdorff"]   # symmetry of the aggregation
        assert O.meanmin_from_dist(DqT) == pytest.approx(c["meanmin_Q_to_target"])
        if "meanmin_target_to_Q" in c:
            assert O.meanmin_from_dist(M) == pytest.approx(c["meanmin_target_to_Q"])
        assert O.min_from_dist(M) == c["min"]
        if "hausdorff_printed_excluded" in c:  # reading R11: Def 4 on the printed matrix gives 1
            assert O.hausdorff_from_dist(DqT) == 1.0


def test_hausdorff_example2():
    g = gold("example2.json")
    Q, V = np.array(g["Q"]), np.array(g["V"])
    D = O.pairwise_dist(Q, V)
    assert D.min(axis=1).tolist() == g["min_over_V_for_each_q"]
    assert D.min(axis=0).tolist() == g["min_over_Q_for_each_v"]
    assert O.hausdorff(Q, V) == g["hausdorff"] == max(g["directed_V_to_Q"], g["directed_Q_to_V"])
    assert O.hausdorff(V, Q) == g["hausdorff"]


def _haus_by_balls(Q, V, iters=60):
    # independent characterisation: the smallest eps with Q in V_eps and V in Q_eps
    D = O.pairwise_dist(Q, V)
    lo, hi = 0.0, float(D.max()) + 1.0
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        covered = all((D[i] <= mid).any() for i in range(D.shape[0])) and \
            all((D[:, j] <= mid).any() for j in range(D.shape[1]))
        lo, hi = (lo, mid) if covered else (mid, hi)
    return hi


def test_hausdorff_metric_properties_and_independent_forms():
    rng = np.random.default_rng(9)
    for trial in range(40):
        d = int(rng.integers(1, 6))
        A, B, C = (rng.standard_normal((int(rng.integers(1, 6)), d)) for _ in range(3))
        hab = O.hausdorff(A, B)
        assert hab == O.hausdorff(B, A)
        assert O.hausdorff(A, A) == 0.0
        assert hab <= O.hausdorff(A, C) + O.hausdorff(C, B) + 1e-12
        D = O.pairwise_dist(A, B)
        assert D.min() <= hab <= D.max()                   # Lemma 1 sandwich (distance form)
        assert hab == pytest.approx(_haus_by_balls(A, B), abs=1e-12)
        assert O.hausdorff_gram(A, B) == pytest.approx(hab, abs=1e-6)
        # explicit loops, no numpy reductions
        dq = max(min(float(np.sqrt(((a - b) ** 2).sum())) for b in B) for a in A)
        dv = max(min(float(np.sqrt(((a - b) ** 2).sum())) for a in A) for b in B)
        assert hab == pytest.approx(max(dq, dv), rel=1e-15)


def test_hausdorff_singletons_closed_form():
    q = np.array([[1.0, 2.0, 2.0]])
    v = np.array([[0.0, 0.0, 0.0]])
    assert O.hausdorff(q, v) == 3.0
    assert O.hausdorff(np.array([[0.0], [4.0]]), np.array([[1.0]])) == 3.0


# ----------------------------------------------------------------- top-k and the whole path

def test_set_distance_point_sets_hand_computed():
    """MeanMin / Min / Hausdorff on 1-D point sets whose distance matrix is
    worked out by hand: Q = {0, 10}, A = {1, 7} -> d(Q,A) = [[1, 7], [9, 3]]:
    MeanMin(Q, A) = (1 + 3) / 2 = 2, Min = 1, Haus = 3 (Def 4);
    MeanMin(A, Q) = (1 + 3) / 2 = 2.  Q = {0, 10}, B = {1, 9, 30}:
    d = [[1, 9, 30], [9, 1, 20]] -> MeanMin(Q, B) = 1, MeanMin(B, Q) = (1 + 1 + 20) / 3,
    Min = 1, Haus = 20 (the asymmetry of §3.2)."""
    Q = np.array([[0.0], [10.0]])
    A = np.array([[1.0], [7.0]])
    B = np.array([[1.0], [9.0], [30.0]])
    assert O.set_distance(Q, A, "meanmin") == 2.0
    assert O.set_distance(A, Q, "meanmin") == 2.0
    assert O.set_distance(Q, A, "min") == 1.0
    assert O.set_distance(Q, A, "hausdorff") == 3.0
    assert O.set_distance(Q, B, "meanmin") == 1.0
    assert O.set_distance(B, Q, "meanmin") == pytest.approx(22.0 / 3.0)
    assert O.set_distance(Q, B, "min") == O.set_distance(B, Q, "min") == 1.0
    assert O.set_distance(Q, B, "hausdorff") == O.set_distance(B, Q, "hausdorff") == 20.0


def test_set_distance_singletons_order_and_brute_force():
    """Singletons: all three metrics reduce to ||q - v|| (Def 4).
    Random sets: Min <= MeanMin <= max_q min_v <= Haus, and MeanMin equals a
    pure-Python double loop."""
    rng = np.random.default_rng(11)
    q, v = rng.normal(size=(1, 5)), rng.normal(size=(1, 5))
    e = float(np.sqrt(((q - v) ** 2).sum()))
    for mt in O.METRICS:
        assert O.set_distance(q, v, mt) == pytest.approx(e, rel=1e-15)
    for _ in range(20):
        Q = rng.normal(size=(rng.integers(1, 6), 3))
        V = rng.normal(size=(rng.integers(1, 6), 3))
        mn, mm, h = (O.set_distance(Q, V, mt) for mt in ("min", "meanmin", "hausdorff"))
        assert mn <= mm + 1e-12 and mm <= h + 1e-12
        loop = 0.0
        for a in Q:
            loop += min(sum((float(a[t]) - float(b[t])) ** 2 for t in range(3)) ** 0.5 for b in V)
        assert mm == pytest.approx(loop / len(Q), rel=1e-12)


def test_top_k_order_and_padding():
    ids, d = O.top_k(np.array([7, 3, 5]), np.array([0.5, 0.5, 0.1]), 5)
    assert ids.tolist() == [5, 3, 7, -1, -1]
    assert d[:3].tolist() == [0.1, 0.5, 0.5] and np.all(np.isinf(d[3:]))


def _tiny_db(seed, n=60, d=16):
    rng = np.random.default_rng(seed)
    sizes = rng.integers(1, 7, n)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    X = rng.standard_normal((off[-1], d)).astype(np.float32)
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    return X, off


@pytest.mark.parametrize("kind", ["binary", "count"])
def test_search_with_T_equal_n_is_bruteforce(kind):
    X, off = _tiny_db(10)
    idx = O.OracleIndex(X, off, m=128, s=4, L=8, seed=3, sketch=kind)
    rng = np.random.default_rng(11)
    for _ in range(4):
        Q = rng.standard_normal((int(rng.integers(1, 5)), 16)).astype(np.float32)
        r_ids, r_d = idx.search(Q, 5, idx.n)
        g_ids, g_d = idx.bruteforce(Q, 5)
        assert r_ids.tolist() == g_ids.tolist() and np.array_equal(r_d, g_d)


def test_query_equal_to_db_set_is_rank1_at_zero():
    X, off = _tiny_db(12)
    idx = O.OracleIndex(X, off, m=128, s=4, L=8, seed=3)
    for j in (0, 17, 59):
        ids, dist = idx.search(idx.set_vectors(j), 3, 10)
        assert ids[0] == j and dist[0] == 0.0


def test_filter_monotone_in_T_and_recall():
    X, off = _tiny_db(13, n=200)
    idx = O.OracleIndex(X, off, m=256, s=4, L=8, seed=5, sketch="count")
    Q = X[off[5]:off[6]]
    prev = set()
    for T in (1, 5, 20, 80, 200):
        cur = set(idx.filter(Q, T).tolist())
        assert prev <= cur and len(cur) == T
        prev = cur
    assert O.recall_at_k(np.array([1, 2, 3]), np.array([3, 2, 1])) == 1.0
    assert O.recall_at_k(np.array([1, 7, -1]), np.array([3, 2, 1])) == pytest.approx(1 / 3)


# ------------------------------------------- BioVSS++ stage-1 gate (Alg 6 lines 1, 3-9; Alg 4)

def test_stage1_positions_hand_built():
    """pi = ArgsortDescending(C_Q), P = the first A; ties -> lower position (reading R27)."""
    CQ = np.array([3, 1, 3, 0, 2])
    assert O.stage1_positions(CQ, 1).tolist() == [0]
    assert O.stage1_positions(CQ, 2).tolist() == [0, 2]
    assert O.stage1_positions(CQ, 3).tolist() == [0, 2, 4]
    assert O.stage1_positions(CQ, 9).tolist() == [0, 2, 4, 1, 3]


def test_stage1_gate_hand_built_and_alg4_loops():
    """F1 = {i : C_i[p] >= M for some p in P} on hand-made counters, against the literal loops of
    Alg 6 over the inverted index of Alg 4 (every (j, c) pair inserted, zeros included, lists sorted by
    descending count)."""
    C = np.array([[0, 5, 0, 5, 5],   # nothing at P = {0, 2}
                  [1, 0, 0, 0, 0],   # count 1 at p = 0
                  [0, 0, 2, 0, 0],   # count 2 at p = 2
                  [3, 0, 1, 0, 0]])  # counts 3 / 1
    P = O.stage1_positions(np.array([3, 1, 3, 0, 2]), 2)
    want = {0: [0, 1, 2, 3], 1: [1, 2, 3], 2: [2, 3], 3: [3], 4: []}
    I = O.inverted_index(C)
    assert [t[1] for t in I[0]] == [3, 1, 0, 0]  # Alg 4 line 8: descending counts
    for M, ids in want.items():
        assert np.flatnonzero(O.stage1_gate(C, P, M)).tolist() == ids
        assert O.stage1_gate_loops(I, P, M).tolist() == ids


def test_stage1_gate_random_loops_nesting_and_binary_equivalence():
    rng = np.random.default_rng(4)
    C = rng.integers(0, 4, size=(60, 32))
    I = O.inverted_index(C)
    CQ = rng.integers(0, 6, size=32)
    for A in (1, 3, 7):
        P = O.stage1_positions(CQ, A)
        for M in (0, 1, 2, 3):
            g = O.stage1_gate(C, P, M)
            assert np.flatnonzero(g).tolist() == O.stage1_gate_loops(I, P, M).tolist()
            # nesting: more lists -> more sets; a higher minimum count -> fewer
            assert np.all(g <= O.stage1_gate(C, O.stage1_positions(CQ, A + 1), M))
            assert np.all(O.stage1_gate(C, P, M + 1) <= g)
        assert O.stage1_gate(C, P, 0).all()  # M = 0: Alg 4 lists every set with its (possibly zero) count
        # M = 1 on the counters == any binary bit set at P (S = (C > 0))
        assert np.array_equal(O.stage1_gate(C, P, 1), O.stage1_gate((C > 0).astype(np.int64), P, 1))


def test_gated_search_reduces_to_open_search_and_filters():
    """A = m, M = 0 opens stage 1 (F1 = D) and the gated search equals Alg 6 without the gate; with the paper's
    defaults (A = 3, M = 1) every returned set passes the gate; |F1| < T returns F1 whole."""
    rng = np.random.default_rng(7)
    V = rng.standard_normal((120, 16)).astype(np.float32)
    off = np.concatenate([[0], np.cumsum(rng.integers(1, 5, size=40))])
    off = off[off <= 120]
    off[-1] = 120
    oi = O.OracleIndex(V, off, 64, 3, 6, 1)
    Q = V[off[3]:off[4]] + 0.01
    a = oi.search(Q, 5, 20)
    b = oi.search_gated(Q, 5, 20, A=64, M=0)
    assert a[0].tolist() == b[0].tolist()
    P = O.stage1_positions(oi.query_counts(Q), 3)
    gate = O.stage1_gate(oi.db_counts(), P, 1)
    f = oi.filter_gated(Q, 1000, 3, 1)
    assert sorted(f.tolist()) == np.flatnonzero(gate).tolist()
    assert all(gate[i] for i in oi.search_gated(Q, 5, 20, 3, 1)[0] if i >= 0)
    # query counts = the fold of the query codes
    assert oi.query_counts(Q).sum() == Q.shape[0] * 6


# ------------------------------------------- BioVSS Alg 2: Hamming-Hausdorff over codes

def _pack(rows):
    return O.pack_bits(np.array([[c == "1" for c in r] + [False] * (32 - len(r)) for r in rows]))


def test_haus_hamming_hand_worked():
    """Haus^H: Def 4 with hamming distance.  Hand-worked on 4-bit codes:
    Q = {1100, 0011}, V = {1010}: hams (2, 2) -> 2;
    Q = {1100}, V = {1100, 0011}: directed q->V = min(0, 4) = 0, V->Q = max(0, 4) = 4 -> 4 (the asymmetric
    case Def 4's outer max exists for)."""
    assert O.haus_hamming(_pack(["1100", "0011"]), _pack(["1010"])) == 2
    assert O.haus_hamming(_pack(["1100"]), _pack(["1100", "0011"])) == 4
    assert O.haus_hamming(_pack(["1100", "0011"]), _pack(["1100", "0011"])) == 0


def test_haus_hamming_metric_identity_and_codes():
    rng = np.random.default_rng(2)
    L, m = 8, 64
    def codes(nv):
        a = rng.standard_normal((nv, m))
        return O.pack_bits(O.wta(a.astype(np.float32), L))
    sets = [codes(int(rng.integers(1, 6))) for _ in range(8)]
    for X in sets:
        for Y in sets:
            h = O.haus_hamming(X, Y)
            assert h == O.haus_hamming(Y, X)                      # symmetric
            # ham = 2L - 2 <h_q, h_v> on codes with exactly L ones
            dots = (O.unpack_bits(X, m).astype(int) @ O.unpack_bits(Y, m).astype(int).T)
            assert np.array_equal(O.hamming_matrix(X, Y), 2 * L - 2 * dots)
            for Z in sets:
                assert O.haus_hamming(X, Z) <= h + O.haus_hamming(Y, Z)  # triangle inequality
        assert O.haus_hamming(X, X) == 0


def test_alg2_search_with_c_equal_n_is_bruteforce():
    rng = np.random.default_rng(9)
    V = rng.standard_normal((90, 12)).astype(np.float32)
    off = np.array([0, 3, 7, 8, 15, 20, 26, 30, 41, 50, 60, 61, 70, 80, 90])
    oi = O.OracleIndex(V, off, 64, 3, 8, 5)
    Q = V[off[4]:off[5]] + 0.02
    n = off.shape[0] - 1
    assert O.top_k(*oi.search_alg2(Q, 4, n), 4)[0].tolist() == oi.bruteforce(Q, 4)[0].tolist()
    cand, dH = O.alg2_candidates(O.encode(Q, oi.W, 8), oi.codes, off, 5)
    assert cand.tolist() == O.select_top_T(dH, 5).tolist() and len(cand) == 5
