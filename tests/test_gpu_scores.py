"""GPU parity of the OVERLAP filter score (reading R24, SURVEY A1 flag) against
the oracle (-m gpu): candidates and keys bit-exact given the GPU sketches
(binary FP4 tensor-core scan on the sampled-threshold and full-key paths, the
count-sketch int8 scan), and the whole search (top-k within 1e-4, ids equal up
to ties)."""
import numpy as np
import pytest

from gen import synth
from oracle import bvss_oracle as O
from tests._common import check_topk, oracle_from_gpu_sketches

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2412_03301_b200.bvss")

CASES = {
    "cfg1": ("cfg1", {}, 0),
    "cfg3-sampled": ("cfg3", dict(n=70001, nq=6, T=300), 0),   # n >= 65536: sampled threshold + fused emission
    "cfg3-full": ("cfg3", dict(n=70001, nq=6, T=300), 1),      # select_mode 1: every key written
    "cfg2s": ("cfg2", dict(n=3001, nq=5, T=200), 0),           # count sketches (int8 tensor-core scan)
}


def _need_gpu():
    if B.device_count() < 1:
        pytest.fail("no sm_100 device visible to libbvss (the GPU tests must run on a B200)")


@pytest.fixture(scope="module", params=list(CASES))
def scase(request):
    _need_gpu()
    name, ov, sel = CASES[request.param]
    cfg = synth.get_config(name, **ov)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = B.Index(data["vectors"], data["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed,
                  score="overlap", select_mode=sel)
    yield dict(cfg=cfg, data=data, idx=idx)
    idx.close()


def _k0(cfg):
    return 2 * cfg.m if cfg.sketch == "binary" else 2 * cfg.m * 255 * 255


def test_overlap_filter_given_gpu_sketches(scase):
    cfg, d, idx = scase["cfg"], scase["data"], scase["idx"]
    db = idx.export_sketches()
    qsk = idx.query_sketch(d["queries"], d["q_offsets"])
    for T in (1, 7, cfg.T, cfg.n + 3):
        cand, score = idx.filter(d["queries"], d["q_offsets"], T)
        for qi in range(cand.shape[0]):
            ov = O.overlap_scores(qsk[qi], db, cfg.sketch)
            ref = O.select_top_T(-ov, T)            # descending overlap, ties by id
            got = cand[qi][cand[qi] >= 0]
            assert got.shape[0] == min(T, cfg.n)
            assert np.all(np.diff(got) > 0)
            assert np.array_equal(np.sort(ref), got)
            assert np.array_equal(score[qi][: got.shape[0]].astype(np.int64), _k0(cfg) - 2 * ov[got])


def test_overlap_search_matches_oracle(scase):
    cfg, d, idx = scase["cfg"], scase["data"], scase["idx"]
    ids, dist = idx.search(d["queries"], d["q_offsets"], cfg.k, cfg.T)
    oi = oracle_from_gpu_sketches(cfg, d, idx, score="overlap")
    V, off = d["vectors"], d["offsets"]
    for qi in range(ids.shape[0]):
        Q = d["queries"][d["q_offsets"][qi]:d["q_offsets"][qi + 1]]
        r_ids, r_d = oi.search(Q, cfg.k, cfg.T)
        check_topk(ids[qi], dist[qi], r_ids, r_d, lambda i: O.hausdorff(Q, V[off[i]:off[i + 1]]))


def test_binarized_count_index_matches_oracle():
    """BINARIZED (R25) on a count-sketch config: the index is a binary one (FP4 scan); its candidates equal
    the oracle's Hamming between binarised count sketches, and the search matches the oracle pipeline."""
    _need_gpu()
    cfg = synth.get_config("cfg2", n=2500, nq=5, T=150)
    d = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = B.Index(d["vectors"], d["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch="count", seed=cfg.seed,
                  score="binarized")
    oi = O.OracleIndex(d["vectors"], d["offsets"], cfg.m, cfg.s, cfg.L, cfg.seed, sketch="count", score="binarized")
    db = idx.export_sketches()
    qsk = idx.query_sketch(d["queries"], d["q_offsets"])
    cand, score = idx.filter(d["queries"], d["q_offsets"], cfg.T)
    for qi in range(cand.shape[0]):
        sc = O.hamming_scores(qsk[qi], db)
        got = cand[qi][cand[qi] >= 0]
        assert np.array_equal(np.sort(O.select_top_T(sc, cfg.T)), got)
        assert np.array_equal(score[qi][: got.shape[0]].astype(np.int64), sc[got])
    ids, dist = idx.search(d["queries"], d["q_offsets"], cfg.k, cfg.T)
    idx.close()
    V, off = d["vectors"], d["offsets"]
    for qi in range(ids.shape[0]):
        Q = d["queries"][d["q_offsets"][qi]:d["q_offsets"][qi + 1]]
        r_ids, r_d = oi.search(Q, cfg.k, cfg.T)
        check_topk(ids[qi], dist[qi], r_ids, r_d, lambda i: O.hausdorff(Q, V[off[i]:off[i + 1]]))


@pytest.mark.parametrize("ov", [dict(n=3001, nq=5, T=200), dict(n=20011, nq=3, T=500, d=64)])
def test_l1_count_score_matches_oracle(ov):
    """L1 (R26) on count sketches: SIMT vabsdiffu4/dp4a scan + full-key select, candidates and keys bit-exact
    given the GPU sketches, and the search against the oracle pipeline."""
    _need_gpu()
    cfg = synth.get_config("cfg2", **ov)
    d = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = B.Index(d["vectors"], d["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch="count", seed=cfg.seed, score="l1")
    db = idx.export_sketches()
    qsk = idx.query_sketch(d["queries"], d["q_offsets"])
    for T in (1, cfg.T, cfg.n + 2):
        cand, score = idx.filter(d["queries"], d["q_offsets"], T)
        for qi in range(cand.shape[0]):
            sc = O.count_l1_scores(qsk[qi], db)
            got = cand[qi][cand[qi] >= 0]
            assert got.shape[0] == min(T, cfg.n)
            assert np.array_equal(np.sort(O.select_top_T(sc, T)), got)
            assert np.array_equal(score[qi][: got.shape[0]].astype(np.int64), sc[got])
    ids, dist = idx.search(d["queries"], d["q_offsets"], cfg.k, cfg.T)
    oi = oracle_from_gpu_sketches(cfg, d, idx, score="l1")
    idx.close()
    V, off = d["vectors"], d["offsets"]
    for qi in range(ids.shape[0]):
        Q = d["queries"][d["q_offsets"][qi]:d["q_offsets"][qi + 1]]
        r_ids, r_d = oi.search(Q, cfg.k, cfg.T)
        check_topk(ids[qi], dist[qi], r_ids, r_d, lambda i: O.hausdorff(Q, V[off[i]:off[i + 1]]))
