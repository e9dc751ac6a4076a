"""Shared helpers for the parity tests (test infrastructure only)."""
import numpy as np

from oracle import bvss_oracle as O

REL = 1e-4     # BJ north_star: Hausdorff distances within 1e-4 relative
ABS = 1e-6     # absolute floor for (near-)zero distances


def dist_close(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) <= np.maximum(REL * np.abs(b), ABS)


def check_topk(gpu_ids, gpu_dist, oracle_ids, oracle_dist, oracle_dist_of):
    """Tie-tolerant top-k comparison: ids equal up to distance ties
    within tolerance, and every returned distance within tolerance of the
    oracle's fp64 distance of that id.  `oracle_dist_of(id)` gives the oracle
    distance of any id."""
    gpu_ids = [int(x) for x in gpu_ids]
    oracle_ids = [int(x) for x in oracle_ids]
    valid = [i for i in oracle_ids if i >= 0]
    if not valid:
        assert all(i < 0 for i in gpu_ids)
        return
    dk = float(oracle_dist[len(valid) - 1])
    lo, hi = dk * (1 - REL) - ABS, dk * (1 + REL) + ABS
    for i in set(gpu_ids) ^ set(oracle_ids):
        if i < 0:
            raise AssertionError(f"padding mismatch: gpu {gpu_ids} oracle {oracle_ids}")
        di = oracle_dist_of(i)
        assert lo <= di <= hi, f"id {i} (oracle dist {di}) differs outside the tie band [{lo}, {hi}]"
    for i, g in zip(gpu_ids, gpu_dist):
        if i < 0:
            assert np.isinf(g)
            continue
        od = oracle_dist_of(i)
        assert dist_close(g, od), f"id {i}: gpu {g} vs oracle {od}"
    # ordering: distances non-decreasing, ties by id
    gd = [float(x) for i, x in zip(gpu_ids, gpu_dist) if i >= 0]
    assert all(gd[j] <= gd[j + 1] for j in range(len(gd) - 1))


def codes_match_modulo_near_ties(gpu_codes, ora_codes, V, W, L, m):
    """Codes bit-exact except rows whose fp64 activation is within 1e-5 of the
    L-th largest (BJ north_star exemption)."""
    diff = np.flatnonzero((gpu_codes != ora_codes).any(axis=1))
    if diff.size == 0:
        return 0
    near = O.near_tie_rows(V[diff], W, L)
    gb = O.unpack_bits(gpu_codes[diff], m)
    ob = O.unpack_bits(ora_codes[diff], m)
    for r in range(diff.size):
        sym = gb[r] ^ ob[r]
        assert np.all(near[r][sym]), f"vector {diff[r]}: code differs on rows that are not near-ties"
    return int(diff.size)


def offsets_from_sizes(sizes):
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


_ORACLES = {}


def oracle_from_gpu_sketches(cfg, data, gpu_idx, score="default"):
    """An oracle index over the GPU's exported database sketches (stage-wise parity: the sketches are
    checked bit-exact elsewhere), cached per workload -- the database encode dominates the oracle time."""
    key = (cfg.name, cfg.n, cfg.nq, cfg.d, cfg.seed, cfg.sketch, score)
    if key not in _ORACLES:
        _ORACLES[key] = O.OracleIndex(data["vectors"], data["offsets"], cfg.m, cfg.s, cfg.L, cfg.seed,
                                      sketch=cfg.sketch, score=score, sketches=gpu_idx.export_sketches())
    return _ORACLES[key]
