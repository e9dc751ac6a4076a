"""Parity at BASELINE.json's full size, in the launch configuration bench.py times (-m gpu).

cfg3 exactly as the bench generates it (n = 1,000,000 sets, d = 384, ~18M database
vectors, 10,000 query sets, k = 10, on the GPU with the same seed), one index, and:

  * the database encode + sketch fold on a random 2000-set sample spread over all
    1M sets, bit-exact against the oracle's own encode (Alg 1 / FlyHash + WTA,
    P:315-335; near-tie rows exempt as everywhere else);
  * K8, the brute force that defines the bench's recall ground truth, on the
    bench's 1000-query recall subset in ONE call: sampled queries against the
    oracle's exact top-k over all 1M sets (Def 4, "precise
    calculations"), tie-tolerant;
  * the timed call itself, bvss_search over the whole 10k batch at T_GATE =
    600,000 (candidate bitmap + dense refine): sampled outputs the oracle can
    compute one by one -- every returned distance equals the oracle's fp64
    Hausdorff of that set, the list is sorted with ties by id, and the j-th
    distance is never below the oracle's exact j-th over all n sets (the search
    ranks a subset of the database; Alg 6).

The oracle brute force over 1M sets runs on the host cores (fork pool over set ranges
of GPU-resident chunks copied to the host); the GPU side never sees oracle output.
"""
import multiprocessing as mp
import os

import numpy as np
import pytest

from gen import synth
from oracle import bvss_oracle as O
from tests._common import ABS, REL, check_topk, dist_close

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2412_03301_b200.bvss")

T_GATE = 600_000        # bench.py T_GATE["cfg3"]
R_SUBSET = 1000         # bench.py --recall-queries default
SAMPLE_Q = (0, 411, 999)  # queries of the recall subset checked against the oracle's brute force
SAMPLE_Q_BATCH = (0, 411, 999, 5003, 9999)  # queries of the timed 10k batch checked one by one

_G = {}  # fork-shared host chunk for the oracle workers


def _bf_worker(rng_):
    lo, hi = rng_
    V, off, base, Qs, k = _G["V"], _G["off"], _G["base"], _G["Qs"], _G["k"]
    out = []
    for Q in Qs:
        ids, d = O.bruteforce_topk(Q, V, off, k, ids=np.arange(lo, hi, dtype=np.int64))
        out.append((ids + base, d))
    return out


def oracle_bruteforce(vec_dev, off_np, Qs, k, chunk_sets=100_000):
    """Exact top-k over all sets for each query of Qs (oracle.bruteforce_topk per set range, merged by
    oracle.top_k)."""
    n = off_np.shape[0] - 1
    cores = os.cpu_count() or 1
    parts = [[] for _ in Qs]
    ctx = mp.get_context("fork")
    for c0 in range(0, n, chunk_sets):
        c1 = min(n, c0 + chunk_sets)
        v0, v1 = int(off_np[c0]), int(off_np[c1])
        _G.update(V=vec_dev[v0:v1].cpu().numpy().astype(np.float64), off=off_np[c0:c1 + 1] - v0, base=c0, Qs=Qs, k=k)
        step = (c1 - c0 + cores - 1) // cores
        with ctx.Pool(cores) as pool:
            res = pool.map(_bf_worker, [(s, min(c1 - c0, s + step)) for s in range(0, c1 - c0, step)])
        for r in res:
            for qi, (ids, d) in enumerate(r):
                parts[qi].append((ids, d))
    _G.clear()
    out = []
    for p in parts:
        ids = np.concatenate([x[0] for x in p])
        d = np.concatenate([x[1] for x in p])
        out.append(O.top_k(ids, d, k))
    return out


class _DevRows:
    """Host rows of a device tensor on demand (the full database never goes to the host at once)."""

    def __init__(self, t):
        self.t = t

    def __getitem__(self, key):
        import torch
        if isinstance(key, slice):
            return self.t[key].cpu().numpy()
        return self.t[torch.as_tensor(np.asarray(key), device=self.t.device)].cpu().numpy()


@pytest.fixture(scope="module")
def full():
    if B.device_count() < 1:
        pytest.fail("no sm_100 device visible to libbvss (the GPU tests must run on a B200)")
    cfg = synth.get_config("cfg3")
    assert cfg.n == 1_000_000 and cfg.nq == 10_000 and cfg.d == 384
    g = synth.generate(cfg, device="cuda")
    idx = B.Index(g["vectors"], g["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed,
                  keep_codes=True)
    yield cfg, g, idx
    idx.close()


def test_fullsize_db_sketches_sample(full):
    from tests.test_gpu_scale import check_db_sketches_sample
    cfg, g, idx = full
    data = {"vectors": _DevRows(g["vectors"]), "offsets": g["offsets"].cpu().numpy()}
    check_db_sketches_sample(cfg, data, idx, nsample=2000, seed=7)


def test_fullsize_k8_and_gated_batch_match_oracle(full):
    cfg, g, idx = full
    k = cfg.k
    qo_all = g["q_offsets"]
    qo_sub = qo_all[: R_SUBSET + 1].contiguous()
    qv_sub = g["queries"][: int(qo_sub[-1])].contiguous()
    gt_ids, gt_d = idx.bruteforce(qv_sub, qo_sub, k)        # K8: the bench's ground-truth call
    ids, dd = idx.search(g["queries"], qo_all, k, T_GATE)    # the bench's timed call (whole batch)
    gt_ids, gt_d, ids, dd = (x.cpu().numpy() for x in (gt_ids, gt_d, ids, dd))

    off = g["offsets"].cpu().numpy()
    qo = qo_all.cpu().numpy()
    qh = g["queries"].cpu().numpy()
    Qs = {qi: qh[qo[qi]:qo[qi + 1]] for qi in sorted(set(SAMPLE_Q) | set(SAMPLE_Q_BATCH))}
    order = sorted(Qs)
    bf = dict(zip(order, oracle_bruteforce(g["vectors"], off, [Qs[q] for q in order], k)))

    def dist_of(Q):
        return lambda i: O.hausdorff(Q, g["vectors"][int(off[i]):int(off[i + 1])].cpu().numpy())

    for qi in SAMPLE_Q:  # K8 == the oracle's exact top-k over all 1M sets
        r_ids, r_d = bf[qi]
        check_topk(gt_ids[qi], gt_d[qi], r_ids, r_d, dist_of(Qs[qi]))
    for qi in SAMPLE_Q_BATCH:  # the gated search: one-by-one distances, order, never better than exact
        f = dist_of(Qs[qi])
        got = [(int(i), float(x)) for i, x in zip(ids[qi], dd[qi]) if i >= 0]
        assert len(got) == k, f"query {qi}: {len(got)} results"
        for i, x in got:
            assert dist_close(x, f(i)), f"query {qi} id {i}: gpu {x} vs oracle {f(i)}"
        assert all((a[1], a[0]) <= (b[1], b[0]) or abs(a[1] - b[1]) <= REL * b[1] + ABS
                   for a, b in zip(got, got[1:])), f"query {qi}: not sorted"
        assert len({i for i, _ in got}) == k
        r_d = bf[qi][1]
        for j in range(k):
            assert got[j][1] >= r_d[j] * (1 - REL) - ABS, f"query {qi} rank {j}: below the exact top-k"
    # the gate's own claim: rank 1 of the sampled recall-subset queries is the exact nearest set
    hit = [ids[qi][0] == bf[qi][0][0] or dist_close(dd[qi][0], bf[qi][1][0]) for qi in SAMPLE_Q]
    assert all(hit), f"rank-1 misses at T={T_GATE}: {hit}"
