"""GPU parity: every stage of the CUDA path against the oracle on the same seeded
inputs (-m gpu).  Each stage is fed the GPU's previous-stage output, so a
legitimate near-tie flip upstream cannot cascade (SURVEY §4 layer 2):
  codes      bit-exact except near-ties (|a - a_(L)| <= 1e-5 |a_(L)|)
  sketches   bit-exact given the GPU codes
  candidates bit-exact (ids and scores) given the GPU sketches
  Hausdorff  tensor-core H^2 within the refine error bound; final top-k within
             1e-4 relative, ids equal up to ties within that tolerance.
"""
import math

import numpy as np
import pytest

from gen import synth
from oracle import bvss_oracle as O
from tests._common import (check_topk, codes_match_modulo_near_ties, dist_close, offsets_from_sizes,
                           oracle_from_gpu_sketches)

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2412_03301_b200.bvss")


def _need_gpu():
    if B.device_count() < 1:
        pytest.fail("no sm_100 device visible to libbvss (the GPU tests must run on a B200)")


# shapes: (config, overrides) -- small n so the oracle finishes in seconds, several
# tiles / warps / CTAs and a ragged tail everywhere
CASES = {
    "cfg1": ("cfg1", {}),
    "cfg2s": ("cfg2", dict(n=3001, nq=6, T=300)),
    "cfg3s": ("cfg3", dict(n=4999, nq=6, T=400)),
    "cfg4s": ("cfg4", dict(n=1999, nq=5, T=300)),
}


@pytest.fixture(scope="module", params=list(CASES))
def case(request):
    _need_gpu()
    name, ov = CASES[request.param]
    cfg = synth.get_config(name, **ov)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = B.Index(data["vectors"], data["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed,
                  keep_codes=True)
    W = O.projection(cfg.seed, cfg.m, cfg.s, cfg.d)
    return dict(cfg=cfg, data=data, idx=idx, W=W)


def test_projection_identical(case):
    assert np.array_equal(case["idx"].export_projection(), case["W"])


def test_codes_bit_exact(case):
    cfg, d = case["cfg"], case["data"]
    V = d["vectors"]
    gpu = case["idx"].export_codes()
    ora = O.encode(V, case["W"], cfg.L)
    ndiff = codes_match_modulo_near_ties(gpu, ora, V, case["W"], cfg.L, cfg.m)
    assert ndiff <= max(1, V.shape[0] // 10000)
    assert np.all(O.popcount_rows(gpu) == cfg.L)


def test_sketches_given_gpu_codes(case):
    cfg, d = case["cfg"], case["data"]
    codes = case["idx"].export_codes()
    gpu = case["idx"].export_sketches()
    if cfg.sketch == "binary":
        ref = O.sketch_binary(codes, d["offsets"])
    else:
        ref = O.sketch_count(codes, d["offsets"], cfg.m)
    assert np.array_equal(gpu, ref)


def test_query_sketches_given_gpu_codes(case):
    cfg, d = case["cfg"], case["data"]
    sk, qcodes = case["idx"].query_sketch(d["queries"], d["q_offsets"], with_codes=True)
    ora = O.encode(d["queries"], case["W"], cfg.L)
    codes_match_modulo_near_ties(qcodes, ora, d["queries"], case["W"], cfg.L, cfg.m)
    if cfg.sketch == "binary":
        assert np.array_equal(sk, O.sketch_binary(qcodes, d["q_offsets"]))
    else:
        assert np.array_equal(sk, O.sketch_count(qcodes, d["q_offsets"], cfg.m))


def _oracle_scores(cfg, qsk, db_sk):
    return O.hamming_scores(qsk, db_sk) if cfg.sketch == "binary" else O.count_l2_scores(qsk, db_sk)


def test_filter_candidates_given_gpu_sketches(case):
    cfg, d, idx = case["cfg"], case["data"], case["idx"]
    db = idx.export_sketches()
    qsk = idx.query_sketch(d["queries"], d["q_offsets"])
    for T in (1, 7, cfg.T, cfg.n, cfg.n + 5):
        cand, score = idx.filter(d["queries"], d["q_offsets"], T)
        for qi in range(cand.shape[0]):
            sc = _oracle_scores(cfg, qsk[qi], db)
            ref = O.select_top_T(sc, T)
            got = cand[qi][cand[qi] >= 0]
            assert got.shape[0] == min(T, cfg.n)
            assert np.all(np.diff(got) > 0), "candidates must come out in ascending id order"
            assert np.array_equal(np.sort(ref), got)
            assert np.array_equal(score[qi][: got.shape[0]], sc[got])


def test_refine_given_gpu_candidates(case):
    cfg, d, idx = case["cfg"], case["data"], case["idx"]
    cand, _ = idx.filter(d["queries"], d["q_offsets"], cfg.T)
    ids, dist, approx = idx.refine(d["queries"], d["q_offsets"], cand, cfg.k)
    V, off = d["vectors"], d["offsets"]
    for qi in range(cand.shape[0]):
        Q = d["queries"][d["q_offsets"][qi]:d["q_offsets"][qi + 1]]
        c = cand[qi][cand[qi] >= 0]
        h = O.refine(Q, c, V, off)
        E = idx.error_bound(math.sqrt(float((Q.astype(np.float64) ** 2).sum(1).max())))
        # tensor-core H^2 within the rigorous bound of the refine arithmetic
        err = np.abs(approx[qi][: c.shape[0]].astype(np.float64) - h * h)
        assert np.all(err <= E), f"max err {err.max()} > bound {E}"
        o_ids, o_d = O.top_k(c, h, cfg.k)
        lookup = dict(zip(c.tolist(), h.tolist()))
        check_topk(ids[qi], dist[qi], o_ids, o_d, lambda i: lookup[i])


def test_search_matches_oracle_pipeline(case):
    cfg, d, idx = case["cfg"], case["data"], case["idx"]
    ids, dist = idx.search(d["queries"], d["q_offsets"], cfg.k, cfg.T)
    oi = O.OracleIndex(d["vectors"], d["offsets"], cfg.m, cfg.s, cfg.L, cfg.seed, sketch=cfg.sketch, W=case["W"])
    V, off = d["vectors"], d["offsets"]
    for qi in range(ids.shape[0]):
        Q = d["queries"][d["q_offsets"][qi]:d["q_offsets"][qi + 1]]
        r_ids, r_d = oi.search(Q, cfg.k, cfg.T)
        check_topk(ids[qi], dist[qi], r_ids, r_d, lambda i: O.hausdorff(Q, V[off[i]:off[i + 1]]))


def test_search_T_equal_n_is_bruteforce(case):
    cfg, d, idx = case["cfg"], case["data"], case["idx"]
    if cfg.n > 5000:
        pytest.skip("brute force oracle too slow")
    nq = 3
    qo = d["q_offsets"][: nq + 1]
    Qall = d["queries"][: qo[-1]]
    ids, dist = idx.search(Qall, qo, cfg.k, cfg.n)
    V, off = d["vectors"], d["offsets"]
    for qi in range(nq):
        Q = Qall[qo[qi]:qo[qi + 1]]
        h = O.refine(Q, np.arange(cfg.n), V, off)
        o_ids, o_d = O.top_k(np.arange(cfg.n), h, cfg.k)
        check_topk(ids[qi], dist[qi], o_ids, o_d, lambda i: h[i])


# ----------------------------------------------------------------- edge cases

def test_edge_shapes_and_degenerate_sets():
    _need_gpu()
    rng = np.random.default_rng(0)
    d, m, s, L = 30, 64, 3, 5   # d not a multiple of 4/8, smallest m, ragged everything
    sizes = np.array([1, 1, 3, 1, 7, 2, 1, 130, 1, 4, 1, 1, 9], dtype=np.int64)  # a set > 128 rows spans tiles
    off = offsets_from_sizes(sizes)
    X = rng.standard_normal((off[-1], d)).astype(np.float32)
    X[off[3]] = X[off[0]]           # duplicate vectors across sets
    X[off[5]:off[6]] = X[off[4]]    # duplicates inside a set
    for kind in ("binary", "count"):
        idx = B.Index(X, off, m=m, s=s, L=L, sketch=kind, seed=9, keep_codes=True)
        W = O.projection(9, m, s, d)
        assert np.array_equal(idx.export_projection(), W)
        codes = idx.export_codes()
        codes_match_modulo_near_ties(codes, O.encode(X, W, L), X, W, L, m)
        # queries: exact copies of DB sets (rank 1 at distance 0), a singleton, the 130-row set
        qsets = [4, 0, 7, 12]
        Q = np.concatenate([X[off[j]:off[j + 1]] for j in qsets])
        qo = offsets_from_sizes([sizes[j] for j in qsets])
        k = 20  # k > n: padding
        ids, dist = idx.search(Q, qo, k, 10_000)  # T > n: clamped -> brute force
        for qi, j in enumerate(qsets):
            Qj = Q[qo[qi]:qo[qi + 1]]
            h = O.refine(Qj, np.arange(len(sizes)), X, off)
            o_ids, o_d = O.top_k(np.arange(len(sizes)), h, k)
            check_topk(ids[qi], dist[qi], o_ids, o_d, lambda i: h[i])
            assert dist[qi][0] == 0.0
            assert ids[qi][len(sizes):].tolist() == [-1] * (k - len(sizes))


def test_L_equals_m_all_ones():
    _need_gpu()
    rng = np.random.default_rng(1)
    X = rng.standard_normal((50, 8)).astype(np.float32)
    off = offsets_from_sizes([5] * 10)
    idx = B.Index(X, off, m=32, s=2, L=32, seed=1, keep_codes=True)
    assert np.all(idx.export_codes() == 0xFFFFFFFF)


def test_errors_are_reported():
    _need_gpu()
    X = np.zeros((4, 8), np.float32)
    with pytest.raises(B.BvssError) as e:
        B.Index(X, np.array([0, 2, 2, 4]), m=32, s=2, L=4)      # empty set
    assert e.value.code == B.EINVAL
    with pytest.raises(B.BvssError):
        B.Index(X, np.array([0, 4]), m=48, s=2, L=4)            # m % 32
    with pytest.raises(B.BvssError):
        B.Index(X, np.array([0, 4]), m=32, s=9, L=4)            # s > d
    Xn = X.copy()
    Xn[1, 1] = np.nan
    with pytest.raises(B.BvssError) as e:
        B.Index(Xn, np.array([0, 4]), m=32, s=2, L=4, validate=True)
    assert e.value.code == B.ENONFINITE
    idx = B.Index(np.random.default_rng(0).standard_normal((4, 8)).astype(np.float32), np.array([0, 4]), m=32, s=2, L=4)
    with pytest.raises(B.BvssError) as e:
        idx.search(X[:2], np.array([0, 2]), 5, 3)                # T < k
    assert e.value.code == B.EINVAL


def test_device_tensors_and_determinism():
    _need_gpu()
    torch = pytest.importorskip("torch")
    cfg = synth.get_config("cfg3", n=3000, nq=8, T=300)
    g = synth.generate(cfg, device="cuda")
    idx = B.Index(g["vectors"], g["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed)
    a_ids, a_d = idx.search(g["queries"], g["q_offsets"], cfg.k, cfg.T)
    b_ids, b_d = idx.search(g["queries"], g["q_offsets"], cfg.k, cfg.T)
    assert torch.equal(a_ids, b_ids) and torch.equal(a_d, b_d)
    h = synth.to_numpy(g)
    c_ids, c_d = idx.search(h["queries"], h["q_offsets"], cfg.k, cfg.T)
    assert np.array_equal(a_ids.cpu().numpy(), c_ids) and np.array_equal(a_d.cpu().numpy(), c_d)


def test_refine_terms_modes_agree():
    _need_gpu()
    cfg = synth.get_config("cfg3", n=2000, nq=5, T=200)
    h = synth.to_numpy(synth.generate(cfg, device="cpu"))
    out = []
    for terms in (1, 3, 255):
        idx = B.Index(h["vectors"], h["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, seed=cfg.seed, refine_terms=terms)
        out.append(idx.search(h["queries"], h["q_offsets"], cfg.k, cfg.T))
    for ids, dist in out[1:]:
        assert np.array_equal(ids, out[0][0])
        assert np.all(dist_close(dist, out[0][1]))


# ------------------------------------------------------ selection strategies

def _modes_agree(cfg, data, Ts, env_cap=None, monkeypatch=None):
    out = {}
    for mode in (1, 2):
        idx = B.Index(data["vectors"], data["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed,
                      select_mode=mode)
        res = []
        for T in Ts:
            ids, dist = idx.search(data["queries"], data["q_offsets"], cfg.k, T)
            res.append((ids, dist, idx.stats()))
        out[mode] = res
        if mode == 1:
            out["oracle"] = oracle_from_gpu_sketches(cfg, data, idx)
        idx.close()
    for (i1, d1, s1), (i2, d2, s2) in zip(out[1], out[2]):
        assert s1["select_batches"] == 0
        assert s2["select_batches"] >= 1
        assert np.array_equal(i1, i2)
        assert np.array_equal(d1, d2)
    return out


@pytest.mark.parametrize("name,ov", [("cfg3", dict(n=40000, nq=7, T=400)), ("cfg2", dict(n=20011, nq=5, T=300))])
def test_sampled_select_equals_full_select(name, ov):
    """select_mode 2 (sampled threshold, fused scan emission) returns exactly what
    select_mode 1 (full key rows) returns, and both match the oracle pipeline."""
    _need_gpu()
    cfg = synth.get_config(name, **ov)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    out = _modes_agree(cfg, data, (cfg.k, cfg.T, 4 * cfg.T))
    ids, dist, st = out[2][1]
    oi = out["oracle"]
    V, off = data["vectors"], data["offsets"]
    for qi in range(3):
        Q = data["queries"][data["q_offsets"][qi]:data["q_offsets"][qi + 1]]
        r_ids, r_d = oi.search(Q, cfg.k, cfg.T)
        check_topk(ids[qi], dist[qi], r_ids, r_d, lambda i: O.hausdorff(Q, V[off[i]:off[i + 1]]))


def test_sampled_select_fallback_on_overflow(monkeypatch):
    """A per-query emission buffer that overflows sends the batch down the full-key
    path; the answer does not change."""
    _need_gpu()
    cfg = synth.get_config("cfg3", n=30000, nq=4, T=300)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    monkeypatch.setenv("BVSS_DEBUG_EMIT_CAP", "16")
    out = _modes_agree(cfg, data, (cfg.T,))
    assert out[2][0][2]["select_fallbacks"] >= 1


@pytest.mark.parametrize("name,ov", [("cfg3", dict(n=7001, nq=300, T=150)), ("cfg2", dict(n=3333, nq=260, T=90, d=64)),
                                     ("cfg4", dict(n=1500, nq=130, T=60, d=64))])
def test_filter_many_query_tiles(name, ov):
    """Several 128-query tiles (ragged), ragged 256-set database tiles, binary and
    count sketches (m = 1024 resident query tile; m = 2048 streamed): candidates
    and scores bit-exact against the oracle given the GPU sketches, for the
    full-key scan and the sampled-threshold fused scan."""
    _need_gpu()
    cfg = synth.get_config(name, **ov)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    for mode in (1, 2):
        idx = B.Index(data["vectors"], data["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed,
                      select_mode=mode)
        db = idx.export_sketches()
        qsk = idx.query_sketch(data["queries"], data["q_offsets"])
        cand, score = idx.filter(data["queries"], data["q_offsets"], cfg.T)
        ids, dist = idx.search(data["queries"], data["q_offsets"], cfg.k, cfg.T)
        st = idx.stats()
        idx.close()
        for qi in range(cand.shape[0]):
            sc = _oracle_scores(cfg, qsk[qi], db)
            ref = np.sort(O.select_top_T(sc, cfg.T))
            got = cand[qi][cand[qi] >= 0]
            assert np.array_equal(ref, got), f"mode {mode} query {qi}"
            assert np.array_equal(score[qi][: got.shape[0]], sc[got])
        if mode == 1:
            base = (ids, dist)
        else:
            assert np.array_equal(ids, base[0]) and np.array_equal(dist, base[1])


@pytest.mark.parametrize("name,ov,limit", [("cfg1", dict(n=600, nq=5), 0), ("cfg3", dict(n=9000, nq=4), 8500),
                                           ("cfg4", dict(n=700, nq=3), 5)])
def test_bruteforce_matches_oracle(name, ov, limit):
    """K8: exact top-k over the first set_limit sets (several 8192-set chunks merged; limit < k pads)."""
    _need_gpu()
    cfg = synth.get_config(name, **ov)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = B.Index(data["vectors"], data["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed)
    ids, dist = idx.bruteforce(data["queries"], data["q_offsets"], cfg.k, set_limit=limit)
    idx.close()
    V, off = data["vectors"], data["offsets"]
    n_lim = cfg.n if limit <= 0 else min(limit, cfg.n)
    for qi in range(ids.shape[0]):
        Q = data["queries"][data["q_offsets"][qi]:data["q_offsets"][qi + 1]]
        r_ids, r_d = O.bruteforce_topk(Q, V, off, cfg.k, ids=np.arange(n_lim, dtype=np.int64))
        check_topk(ids[qi], dist[qi], r_ids, r_d, lambda i: O.hausdorff(Q, V[off[i]:off[i + 1]]))
        if n_lim < cfg.k:
            assert np.all(ids[qi][n_lim:] == -1) and np.all(np.isinf(dist[qi][n_lim:]))


@pytest.mark.parametrize("rng_sets", ["0", "1500"])
def test_search_range_major_refine(monkeypatch, rng_sets):
    """The refine's range-major group mode (developer switch BVSS_REFINE_GROUP=1: 4 queries per tile,
    candidate lists cut by database range) against the query-major mode and the oracle pipeline, on the
    sampled-threshold search path (n >= 65536, candidate lists sorted by select_buf)."""
    _need_gpu()
    cfg = synth.get_config("cfg3", n=70000, nq=24, T=300)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = B.Index(data["vectors"], data["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed)
    if rng_sets != "0":
        monkeypatch.setenv("BVSS_REFINE_RANGE", rng_sets)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("BVSS_REFINE_GROUP", mode)
        ids, dist = idx.search(data["queries"], data["q_offsets"], cfg.k, cfg.T)
        out[mode] = (ids, dist, idx.stats())
    oi = oracle_from_gpu_sketches(cfg, data, idx)
    idx.close()
    assert out["1"][2]["select_batches"] >= 1
    assert np.array_equal(out["0"][0], out["1"][0]) and np.array_equal(out["0"][1], out["1"][1])
    assert out["0"][2]["fixup_sets"] == out["1"][2]["fixup_sets"]  # identical tensor-core values
    V, off = data["vectors"], data["offsets"]
    ids, dist = out["1"][0], out["1"][1]
    for qi in range(0, cfg.nq, 6):
        Q = data["queries"][data["q_offsets"][qi]:data["q_offsets"][qi + 1]]
        r_ids, r_d = oi.search(Q, cfg.k, cfg.T)
        check_topk(ids[qi], dist[qi], r_ids, r_d, lambda i: O.hausdorff(Q, V[off[i]:off[i + 1]]))


def test_streaming_build_equals_build():
    """bvss_index_begin / append (uneven chunks) / finish builds the same index as bvss_build_index:
    identical codes, sketches and search results; search before finish and over-long appends fail."""
    _need_gpu()
    cfg = synth.get_config("cfg3", n=3001, nq=5, T=200)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    V, off = data["vectors"], data["offsets"]
    kw = dict(m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed, keep_codes=True)
    ref = B.Index(V, off, **kw)
    cuts = [0, 1, 700, 2999, cfg.n]

    def chunks():
        for a, b in zip(cuts, cuts[1:]):
            yield V[off[a]:off[b]], off[a:b + 1] - off[a]
    idx = B.Index.from_chunks(chunks(), n_total=cfg.n, nvec_total=int(off[-1]), d=cfg.d, **kw)
    assert np.array_equal(idx.export_codes(), ref.export_codes())
    assert np.array_equal(idx.export_sketches(), ref.export_sketches())
    r1 = ref.search(data["queries"], data["q_offsets"], cfg.k, cfg.T)
    r2 = idx.search(data["queries"], data["q_offsets"], cfg.k, cfg.T)
    assert np.array_equal(r1[0], r2[0]) and np.array_equal(r1[1], r2[1])
    ref.close()
    idx.close()
    with pytest.raises(B.BvssError) as e:  # more data than declared
        B.Index.from_chunks(chunks(), n_total=cfg.n - 1, nvec_total=int(off[-1]), d=cfg.d, **kw)
    assert e.value.code == B.EINVAL
