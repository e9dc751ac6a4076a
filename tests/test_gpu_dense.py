"""GPU parity of the candidate-major (dense) refine, dense.cu (-m gpu).

The dense kernel computes every (query set, database set) Gram on the tensor
cores with the query tile stationary, prunes by the lower bound
A = max_q min_v D^2 against a running k-th upper bound, and hands the emitted
lists to the exact fp32 fix-up (K6).  Its result must be the exact top-k by
Def 4: identical to the query-major path (both end in the same
exact fp32 recomputation) and within the tie-tolerant rule of the oracle.
Covered: brute force (K8, T = n) with and without a set limit, large-T search
restricted by the candidate bitmap (Alg 6 F2), database sets of more
than 256 rows (exact path), a forced candidate-list overflow (fallback to the
query-major path), d not a multiple of 64, query sets of 1..32 rows packed
into warp bins, and many query tiles (ragged).
"""
import numpy as np
import pytest

from gen import synth
from oracle import bvss_oracle as O
from tests._common import check_topk, offsets_from_sizes, oracle_from_gpu_sketches

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2412_03301_b200.bvss")


def _need_gpu():
    if B.device_count() < 1:
        pytest.fail("no sm_100 device visible to libbvss (the GPU tests must run on a B200)")


def _index(cfg, data, **kw):
    return B.Index(data["vectors"], data["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed,
                   **kw)


@pytest.mark.parametrize("name,ov,limit", [("cfg1", dict(n=1000, nq=10), 0),
                                           ("cfg3", dict(n=6000, nq=300, d=384), 0),
                                           ("cfg3", dict(n=5003, nq=40), 3001),
                                           ("cfg1", dict(n=900, nq=7, d=30), 0)])
def test_dense_bruteforce_matches_oracle(name, ov, limit):
    _need_gpu()
    cfg = synth.get_config(name, **ov)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = _index(cfg, data)
    ids, dist = idx.bruteforce(data["queries"], data["q_offsets"], cfg.k, set_limit=limit)
    st = idx.stats()
    assert st["dense_batches"] == 1, "brute force must run on the dense kernel"
    idx.close()
    V, off = data["vectors"], data["offsets"]
    n_lim = cfg.n if limit <= 0 else limit
    for qi in list(range(0, ids.shape[0], max(1, ids.shape[0] // 6)))[:6]:
        Q = data["queries"][data["q_offsets"][qi]:data["q_offsets"][qi + 1]]
        h = O.refine(Q, np.arange(n_lim), V, off)
        o_ids, o_d = O.top_k(np.arange(n_lim), h, cfg.k)
        check_topk(ids[qi], dist[qi], o_ids, o_d, lambda i: h[i])


@pytest.mark.parametrize("sched", [{}, {"BVSS_DENSE_TPR": "3"}, {"BVSS_DENSE_TPR": "16"},
                                   {"BVSS_DENSE_DYN": "0"}, {"BVSS_DENSE_DYN": "0", "BVSS_DENSE_R": "7"}])
def test_dense_bruteforce_equals_query_major_refine(sched, monkeypatch):
    """Every query: the dense brute force and the query-major refine over all n candidates (bvss_refine) give
    identical ids and distances (the same exact fp32 fix-up decides both).  Under every schedule: the default
    (dynamic range-major units; one range at this n), small ranges (many units per query tile pair: the
    running tau and the list inheritance from the previous range are exercised), the static pair-major
    schedule with its union over ranges."""
    _need_gpu()
    for k, v in sched.items():
        monkeypatch.setenv(k, v)
    cfg = synth.get_config("cfg3", n=3000, nq=200)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = _index(cfg, data)
    ids, dist = idx.bruteforce(data["queries"], data["q_offsets"], cfg.k)
    st = idx.stats()
    assert st["dense_batches"] == 1
    assert 0 < st["dense_survivors"] <= cfg.nq * cfg.n  # (small n: the bound lists fill late, the prune is weak)
    cand = np.tile(np.arange(cfg.n, dtype=np.int32), (cfg.nq, 1))
    r_ids, r_d, _ = idx.refine(data["queries"], data["q_offsets"], cand, cfg.k)
    np.testing.assert_array_equal(ids, r_ids)
    np.testing.assert_array_equal(dist, r_d)
    idx.close()


@pytest.mark.parametrize("T", [1500, 9000])
def test_dense_search_large_T_matches_oracle(T, monkeypatch):
    """Search with a candidate budget that is a large fraction of n goes through the candidate bitmap + dense
    kernel and matches the oracle pipeline (filter to T, exact Hausdorff, top-k)."""
    _need_gpu()
    cfg = synth.get_config("cfg3", n=9000, nq=60, T=T)
    _large_T_case(cfg, T)


@pytest.mark.parametrize("tpr", ["1024", "2"])
def test_dense_search_tiny_sets_bitmap(tpr, monkeypatch):
    """cfg1's sets of 2-8 vectors put up to ~100 sets in one 240-row tile, so the kernel's two prefetched
    bitmap words do not cover every set of a tile and the direct word reads run; 2-tile ranges (many units,
    inheritance) as well as the default."""
    _need_gpu()
    monkeypatch.setenv("BVSS_DENSE_TPR", tpr)
    cfg = synth.get_config("cfg1", n=2000, nq=30, T=700)
    _large_T_case(cfg, 700)


def _large_T_case(cfg, T):
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = _index(cfg, data, select_mode=1)
    ids, dist = idx.search(data["queries"], data["q_offsets"], cfg.k, T)
    st = idx.stats()
    assert st["dense_batches"] == 1
    oi = oracle_from_gpu_sketches(cfg, data, idx)
    V, off = data["vectors"], data["offsets"]
    for qi in range(0, cfg.nq, 7):
        Q = data["queries"][data["q_offsets"][qi]:data["q_offsets"][qi + 1]]
        r_ids, r_d = oi.search(Q, cfg.k, T)
        check_topk(ids[qi], dist[qi], r_ids, r_d, lambda i: O.hausdorff(Q, V[off[i]:off[i + 1]]))
    # the same candidates through the query-major refine: identical
    cand, _ = idx.filter(data["queries"], data["q_offsets"], T)
    r_ids, r_d, _ = idx.refine(data["queries"], data["q_offsets"], cand, cfg.k)
    np.testing.assert_array_equal(ids, r_ids)
    np.testing.assert_array_equal(dist, r_d)
    idx.close()


def test_dense_overflow_falls_back(monkeypatch):
    """A candidate list that overflows its capacity (forced) sends the batch down the query-major path."""
    _need_gpu()
    cfg = synth.get_config("cfg3", n=2500, nq=30)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = _index(cfg, data)
    ids, dist = idx.bruteforce(data["queries"], data["q_offsets"], cfg.k)
    monkeypatch.setenv("BVSS_DEBUG_DENSE_CAP", "8")
    ids2, dist2 = idx.bruteforce(data["queries"], data["q_offsets"], cfg.k)
    assert idx.stats()["dense_batches"] == 0
    np.testing.assert_array_equal(ids, ids2)
    np.testing.assert_array_equal(dist, dist2)
    idx.close()


def test_dense_with_sets_over_256_rows():
    _need_gpu()
    rng = np.random.default_rng(11)
    d = 64
    Q = rng.standard_normal((5, d)).astype(np.float32)
    sets = [rng.standard_normal((int(rng.integers(1, 40)), d)).astype(np.float32) for _ in range(300)]
    sets[17] = np.concatenate([Q[np.arange(300) % 5] + 0.01 * rng.standard_normal((300, d)).astype(np.float32)])
    sets[230] = 2.0 + rng.standard_normal((400, d)).astype(np.float32)
    sets[5] = Q + 0.05 * rng.standard_normal((5, d)).astype(np.float32)
    X = np.concatenate(sets).astype(np.float32)
    off = offsets_from_sizes([s.shape[0] for s in sets])
    n = len(sets)
    qsets = [Q, Q[:3], sets[40][:1]]
    Qa = np.concatenate(qsets).astype(np.float32)
    qo = offsets_from_sizes([q.shape[0] for q in qsets])
    idx = B.Index(X, off, m=256, s=4, L=16, seed=2)
    k = 8
    ids, dist = idx.bruteforce(Qa, qo, k)
    assert idx.stats()["dense_batches"] == 1
    for qi, Qs in enumerate(qsets):
        h = O.refine(Qs, np.arange(n), X, off)
        o_ids, o_d = O.top_k(np.arange(n), h, k)
        check_topk(ids[qi], dist[qi], o_ids, o_d, lambda i: h[i])
    assert ids[0][0] in (5, 17) and ids[0][1] in (5, 17)
    idx.close()
