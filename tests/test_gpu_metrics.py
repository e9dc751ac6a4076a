"""GPU parity of the MeanMin / Min rerank metrics (SURVEY §8(f)
NEXT 4) against the oracle (-m gpu): the refine's tensor-core values within the
error bound of its arithmetic, and the exact top-k within 1e-4 relative, ids
equal up to ties, for query sets on both sides of the 32-row TMEM lane quarter
(cfg2: sets of 1..64 vectors), on the search, refine, brute-force and
exact-only (refine_terms=255) paths."""
import math

import numpy as np
import pytest

from gen import synth
from oracle import bvss_oracle as O
from tests._common import check_topk

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2412_03301_b200.bvss")

CASES = {
    "cfg1": ("cfg1", {}),
    "cfg2s": ("cfg2", dict(n=2001, nq=6, T=200)),
    "cfg3s": ("cfg3", dict(n=3001, nq=5, T=300)),
}


def _need_gpu():
    if B.device_count() < 1:
        pytest.fail("no sm_100 device visible to libbvss (the GPU tests must run on a B200)")


@pytest.fixture(scope="module", params=[(c, mt) for c in CASES for mt in ("meanmin", "min")],
                ids=lambda p: f"{p[0]}-{p[1]}")
def mcase(request):
    _need_gpu()
    cname, metric = request.param
    name, ov = CASES[cname]
    cfg = synth.get_config(name, **ov)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    idx = B.Index(data["vectors"], data["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed,
                  metric=metric)
    yield dict(cfg=cfg, data=data, idx=idx, metric=metric)
    idx.close()


def _Q(d, qi):
    return d["queries"][d["q_offsets"][qi]:d["q_offsets"][qi + 1]]


def test_refine_metric_given_gpu_candidates(mcase):
    cfg, d, idx, mt = mcase["cfg"], mcase["data"], mcase["idx"], mcase["metric"]
    cand, _ = idx.filter(d["queries"], d["q_offsets"], cfg.T)
    ids, dist, approx = idx.refine(d["queries"], d["q_offsets"], cand, cfg.k)
    V, off = d["vectors"], d["offsets"]
    for qi in range(cand.shape[0]):
        Q = _Q(d, qi)
        c = cand[qi][cand[qi] >= 0]
        h = O.refine(Q, c, V, off, mt)
        E = idx.error_bound(math.sqrt(float((Q.astype(np.float64) ** 2).sum(1).max())))
        if mt == "meanmin":  # the tensor-core value is a distance: each row term within sqrt(E)
            err = np.abs(approx[qi][: c.shape[0]].astype(np.float64) - h)
            bound = math.sqrt(E) * (1 + 1e-4) + 1e-5 * h.max()
        else:                # squared distance within E
            err = np.abs(approx[qi][: c.shape[0]].astype(np.float64) - h * h)
            bound = E
        assert np.all(err <= bound), f"max err {err.max()} > bound {bound}"
        o_ids, o_d = O.top_k(c, h, cfg.k)
        lookup = dict(zip(c.tolist(), h.tolist()))
        check_topk(ids[qi], dist[qi], o_ids, o_d, lambda i: lookup[i])


def test_search_metric_matches_oracle(mcase):
    cfg, d, idx, mt = mcase["cfg"], mcase["data"], mcase["idx"], mcase["metric"]
    ids, dist = idx.search(d["queries"], d["q_offsets"], cfg.k, cfg.T)
    oi = O.OracleIndex(d["vectors"], d["offsets"], cfg.m, cfg.s, cfg.L, cfg.seed, sketch=cfg.sketch)
    V, off = d["vectors"], d["offsets"]
    for qi in range(ids.shape[0]):
        Q = _Q(d, qi)
        r_ids, r_d = oi.search(Q, cfg.k, cfg.T, metric=mt)
        check_topk(ids[qi], dist[qi], r_ids, r_d, lambda i: O.set_distance(Q, V[off[i]:off[i + 1]], mt))


@pytest.mark.parametrize("metric", ["meanmin", "min"])
def test_bruteforce_and_exact_mode_metric(metric):
    """K8 with the alternative metric, and the exact-only refine (refine_terms=255) on the same queries."""
    _need_gpu()
    cfg = synth.get_config("cfg2", n=700, nq=4, T=60, d=64)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    V, off = data["vectors"], data["offsets"]
    for terms in (0, 255):
        idx = B.Index(V, off, m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed, metric=metric,
                      refine_terms=terms)
        ids, dist = idx.bruteforce(data["queries"], data["q_offsets"], cfg.k)
        s_ids, s_dist = idx.search(data["queries"], data["q_offsets"], cfg.k, cfg.n)  # T = n: brute force
        idx.close()
        for qi in range(ids.shape[0]):
            Q = _Q(data, qi)
            h = O.refine(Q, np.arange(cfg.n), V, off, metric)
            r_ids, r_d = O.top_k(np.arange(cfg.n), h, cfg.k)
            check_topk(ids[qi], dist[qi], r_ids, r_d, lambda i: h[i])
            check_topk(s_ids[qi], s_dist[qi], r_ids, r_d, lambda i: h[i])


def test_metric_degenerate_cases():
    """A query equal to a database set is at distance 0 under every metric; singleton sets give
    ||q - v|| under every metric; Min <= MeanMin <= Hausdorff on the returned distances."""
    _need_gpu()
    rng = np.random.default_rng(5)
    d = 40
    sizes = [1, 3, 1, 7, 33, 2, 1, 5]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    V = rng.normal(size=(off[-1], d)).astype(np.float32)
    Q = V[off[4]:off[5]].copy()  # the 33-vector set: two TMEM lane quarters
    qo = np.array([0, Q.shape[0]], dtype=np.int64)
    out = {}
    for mt in ("hausdorff", "meanmin", "min"):
        idx = B.Index(V, off, m=64, s=4, L=6, seed=3, metric=mt)
        ids, dist = idx.search(Q, qo, 8, 8)
        idx.close()
        assert ids[0][0] == 4 and dist[0][0] == 0.0
        for i, g in zip(ids[0], dist[0]):
            od = O.set_distance(Q, V[off[i]:off[i + 1]], mt)
            assert abs(g - od) <= max(1e-4 * od, 1e-6), (mt, i, g, od)
        out[mt] = dict(zip(ids[0].tolist(), dist[0].tolist()))
    for i in range(len(sizes)):
        assert out["min"][i] <= out["meanmin"][i] * (1 + 1e-5) + 1e-6
        assert out["meanmin"][i] <= out["hausdorff"][i] * (1 + 1e-5) + 1e-6
    q1 = V[off[0]:off[1]]  # singleton query against singleton sets: all metrics equal ||q - v||
    for mt in ("meanmin", "min"):
        idx = B.Index(V, off, m=64, s=4, L=6, seed=3, metric=mt)
        ids, dist = idx.search(q1, np.array([0, 1], dtype=np.int64), 8, 8)
        idx.close()
        for i, g in zip(ids[0], dist[0]):
            if sizes[i] == 1:
                e = float(np.sqrt(((q1[0].astype(np.float64) - V[off[i]].astype(np.float64)) ** 2).sum()))
                assert abs(g - e) <= max(1e-4 * e, 1e-6)


def test_metric_param_validation():
    _need_gpu()
    V = np.ones((3, 8), dtype=np.float32)
    off = np.array([0, 1, 3], dtype=np.int64)
    p = B.Params(m=32, s=2, L=4, sketch=0, seed=0, projection=None, device=0, flags=0, query_batch=0, refine_terms=0,
                 select_mode=0, metric=7)
    import ctypes as C
    h = C.c_void_p()
    rc = B.lib.bvss_build_index(C.c_void_p(V.ctypes.data), C.c_void_p(off.ctypes.data), 2, 8, C.byref(p), C.byref(h))
    assert rc == -1 and "metric" in B.lib.bvss_last_error().decode()
