"""GPU parity of the candidate-generation variants (gate.cu, -m gpu):

  * BioVSS++ stage 1 (Alg 6 lines 1, 3-9; Alg 4's inverted index):
    the query's A largest count positions, sets with C_i[p] >= M at one of them;
    candidates = the first T of F1 by (score, id), F1 whole when |F1| < T;
  * BioVSS Alg 2: Haus^H over the per-vector codes ranks every set,
    the c = T smallest (ties by id) are refined.

Stage-wise like the other parity tests: the oracle gets the GPU's database
sketches / codes and the GPU's query codes, so candidates and scores are
compared bit for bit; the searches are compared with the tie-tolerant rule.
"""
import numpy as np
import pytest

from gen import synth
from oracle import bvss_oracle as O
from tests._common import check_topk

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2412_03301_b200.bvss")


def _need_gpu():
    if B.device_count() < 1:
        pytest.fail("no sm_100 device visible to libbvss (the GPU tests must run on a B200)")


def _db_counts(cfg, sk):
    return np.asarray(sk, dtype=np.int64) if cfg.sketch == "count" else O.unpack_bits(sk, cfg.m).astype(np.int64)


def _scores(cfg, qsk, db):
    return O.hamming_scores(qsk, db) if cfg.sketch == "binary" else O.count_l2_scores(qsk, db)


@pytest.mark.parametrize("name,ov,A,M", [("cfg3", dict(n=4001, nq=7, T=300), 3, 1),
                                         ("cfg3", dict(n=3001, nq=5, T=300), 1, 1),
                                         ("cfg2", dict(n=3001, nq=6, T=200, d=64), 3, 2),
                                         ("cfg1", dict(n=1000, nq=10), 2, 1)])
def test_gated_filter_bit_exact(name, ov, A, M):
    _need_gpu()
    cfg = synth.get_config(name, **ov)
    d = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = B.Index(d["vectors"], d["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed,
                  gate_A=A, gate_M=M)
    db = idx.export_sketches()
    C = _db_counts(cfg, db)
    qsk, qcodes = idx.query_sketch(d["queries"], d["q_offsets"], with_codes=True)
    qo = d["q_offsets"]
    for T in (cfg.T, cfg.n):  # T = n: every set of F1 (|F1| < T)
        cand, score = idx.filter(d["queries"], qo, T)
        for qi in range(cand.shape[0]):
            CQ = O.sketch_count(qcodes[qo[qi]:qo[qi + 1]], np.array([0, qo[qi + 1] - qo[qi]]), cfg.m)[0]
            P = O.stage1_positions(CQ, A)
            gate = O.stage1_gate(C, P, M)
            sc = _scores(cfg, qsk[qi], db)
            ids = np.flatnonzero(gate)
            ref = np.sort(ids[np.lexsort((ids, sc[ids]))][:T])
            got = cand[qi][cand[qi] >= 0]
            assert np.array_equal(got, ref), f"T={T} query {qi}: {len(got)} vs {len(ref)}"
            assert np.array_equal(score[qi][: got.shape[0]], sc[got])
            if T == cfg.n:
                assert got.shape[0] == gate.sum()
    idx.close()


def test_gated_search_matches_oracle_and_open_gate():
    _need_gpu()
    cfg = synth.get_config("cfg3", n=3001, nq=6, T=250)
    d = synth.to_numpy(synth.generate(cfg, device="cpu"))
    V, off = d["vectors"], d["offsets"]
    idx = B.Index(V, off, m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed, gate_A=3, gate_M=1)
    ids, dist = idx.search(d["queries"], d["q_offsets"], cfg.k, cfg.T)
    oi = O.OracleIndex(V, off, cfg.m, cfg.s, cfg.L, cfg.seed, sketch=cfg.sketch, sketches=idx.export_sketches())
    for qi in range(cfg.nq):
        Q = d["queries"][d["q_offsets"][qi]:d["q_offsets"][qi + 1]]
        r_ids, r_d = oi.search_gated(Q, cfg.k, cfg.T, 3, 1)
        check_topk(ids[qi], dist[qi], r_ids, r_d, lambda i: O.hausdorff(Q, V[off[i]:off[i + 1]]))
    idx.close()
    # M = 0 opens the gate (Alg 4 lists every set, zero counts included): the plain filter
    open_idx = B.Index(V, off, m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed, gate_A=3, gate_M=0)
    plain = B.Index(V, off, m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed, select_mode=1)
    a = open_idx.filter(d["queries"], d["q_offsets"], cfg.T)
    b = plain.filter(d["queries"], d["q_offsets"], cfg.T)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    open_idx.close()
    plain.close()


def test_gated_dense_large_T_equals_query_major():
    """The gate inside the candidate bitmap of the dense refine (large T) gives the query-major result."""
    _need_gpu()
    cfg = synth.get_config("cfg3", n=6000, nq=40, T=3000)
    d = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = B.Index(d["vectors"], d["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed,
                  gate_A=3, gate_M=1)
    ids, dist = idx.search(d["queries"], d["q_offsets"], cfg.k, cfg.T)
    assert idx.stats()["dense_batches"] == 1
    cand, _ = idx.filter(d["queries"], d["q_offsets"], cfg.T)
    r_ids, r_d, _ = idx.refine(d["queries"], d["q_offsets"], cand, cfg.k)
    np.testing.assert_array_equal(ids, r_ids)
    np.testing.assert_array_equal(dist, r_d)
    idx.close()


def test_gate_parameter_errors():
    _need_gpu()
    X = np.random.default_rng(0).standard_normal((40, 8)).astype(np.float32)
    off = np.arange(0, 41, 4)
    with pytest.raises(B.BvssError) as e:
        B.Index(X, off, m=64, s=2, L=4, gate_A=3, gate_M=2)  # binary index: no counts
    assert e.value.code == B.EINVAL
    with pytest.raises(B.BvssError):
        B.Index(X, off, m=64, s=2, L=4, gate_A=65, gate_M=1)


@pytest.mark.parametrize("name,ov", [("cfg3", dict(n=2501, nq=5, T=200)), ("cfg1", dict(n=800, nq=6, T=60)),
                                     ("cfg2", dict(n=1200, nq=4, T=100, d=64))])
def test_alg2_candidates_bit_exact(name, ov):
    """Alg 2 lines 6-9: Haus^H of every set from the per-vector codes, the T smallest by (Haus^H, id)."""
    _need_gpu()
    cfg = synth.get_config(name, **ov)
    d = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = B.Index(d["vectors"], d["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed,
                  filter="alg2")
    codes = idx.export_codes()
    _, qcodes = idx.query_sketch(d["queries"], d["q_offsets"], with_codes=True)
    qo = d["q_offsets"]
    cand, score = idx.filter(d["queries"], qo, cfg.T)
    for qi in range(cand.shape[0]):
        ref, dH = O.alg2_candidates(qcodes[qo[qi]:qo[qi + 1]], codes, d["offsets"], cfg.T)
        got = cand[qi][cand[qi] >= 0]
        assert np.array_equal(got, np.sort(ref))
        assert np.array_equal(score[qi][: got.shape[0]], dH[got])
    idx.close()


def test_alg2_search_matches_oracle():
    _need_gpu()
    cfg = synth.get_config("cfg3", n=2000, nq=5, T=150)
    d = synth.to_numpy(synth.generate(cfg, device="cpu"))
    V, off = d["vectors"], d["offsets"]
    idx = B.Index(V, off, m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed, filter="alg2")
    ids, dist = idx.search(d["queries"], d["q_offsets"], cfg.k, cfg.T)
    oi = O.OracleIndex(V, off, cfg.m, cfg.s, cfg.L, cfg.seed, sketch=cfg.sketch)
    for qi in range(cfg.nq):
        Q = d["queries"][d["q_offsets"][qi]:d["q_offsets"][qi + 1]]
        r_ids, r_d = oi.search_alg2(Q, cfg.k, cfg.T)
        check_topk(ids[qi], dist[qi], r_ids, r_d, lambda i: O.hausdorff(Q, V[off[i]:off[i + 1]]))
    # c = n: brute force
    ids2, dist2 = idx.search(d["queries"], d["q_offsets"], cfg.k, cfg.n)
    bf_ids, bf_d = idx.bruteforce(d["queries"], d["q_offsets"], cfg.k)
    np.testing.assert_array_equal(ids2, bf_ids)
    idx.close()
