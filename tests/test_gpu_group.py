"""The single-process multi-device index (bvss_group_*, include/bvss.h) on the GPU.

Only one B200 is available to this build, so the shards share cuda:0 (devices = [0, 0] / [0, 0, 0]):
the protocol, the in-process collectives (peer copies, histogram sum kernel, K7 merge) and the concurrent
per-shard phases all run; NVLink itself is not exercised.  The merged top-k must equal one index over the
whole database exactly (same kernels on every (query, set) pair, the global top-T by the exact tie
protocol: Alg 6 lines 10-23, with one budget T), and match the oracle pipeline."""
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


def _kw(cfg):
    return dict(m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed)


@pytest.mark.parametrize("devices,cfg_kw", [([0, 0], dict(name="cfg3", n=6001, nq=9, T=300)),
                                            ([0, 0, 0], dict(name="cfg2", n=3001, nq=5, T=120, d=64)),
                                            ([0, 0], dict(name="cfg1", n=500, nq=6, T=600)),
                                            ([0, 0, 0, 0], dict(name="cfg3", n=4003, nq=7, T=3000))])
def test_group_equals_single_index(devices, cfg_kw):
    """(The last case, T = 3000 of 4003 sets, takes the dense candidate-major refine on every shard.)"""
    _need_gpu()
    cfg = synth.get_config(**cfg_kw)
    h = synth.to_numpy(synth.generate(cfg, device="cpu"))
    grp = B.Group(h["vectors"], h["offsets"], devices=devices, **_kw(cfg))
    assert grp.shards == len(devices)
    ids, dist = grp.search(h["queries"], h["q_offsets"], cfg.k, cfg.T)
    bases = [grp.shard_stats(i)[0] for i in range(grp.shards)]
    assert bases[0] == 0 and all(b < c for b, c in zip(bases, bases[1:]))
    grp.close()
    idx = B.Index(h["vectors"], h["offsets"], select_mode=1, **_kw(cfg))
    ref_ids, ref_d = idx.search(h["queries"], h["q_offsets"], cfg.k, cfg.T)
    idx.close()
    np.testing.assert_array_equal(ids, ref_ids)
    np.testing.assert_array_equal(dist, ref_d)


def test_group_matches_oracle():
    _need_gpu()
    cfg = synth.get_config("cfg3", n=4001, nq=6, T=250)
    h = synth.to_numpy(synth.generate(cfg, device="cpu"))
    grp = B.Group(h["vectors"], h["offsets"], devices=[0, 0], **_kw(cfg))
    ids, dist = grp.search(h["queries"], h["q_offsets"], cfg.k, cfg.T)
    grp.close()
    oi = O.OracleIndex(h["vectors"], h["offsets"], cfg.m, cfg.s, cfg.L, cfg.seed, sketch=cfg.sketch)
    V, off = h["vectors"], h["offsets"]
    for qi in range(cfg.nq):
        Q = h["queries"][h["q_offsets"][qi]:h["q_offsets"][qi + 1]]
        r_ids, r_d = oi.search(Q, cfg.k, cfg.T)
        check_topk(ids[qi], dist[qi], r_ids, r_d, lambda i: O.hausdorff(Q, V[off[i]:off[i + 1]]))


def test_group_edge_cases():
    """n < P shrinks the group to n shards; k > n pads with (-1, +inf); bad arguments fail loudly."""
    _need_gpu()
    rng = np.random.default_rng(5)
    V = rng.standard_normal((5, 64)).astype(np.float32)
    off = np.array([0, 2, 5], np.int64)
    grp = B.Group(V, off, devices=[0, 0, 0], m=512, s=6, L=16)
    assert grp.shards == 2
    ids, dist = grp.search(V[:2], np.array([0, 2], np.int64), 4, 10)
    assert ids[0, 0] == 0 and dist[0, 0] == 0.0
    assert list(ids[0, 2:]) == [-1, -1] and np.isinf(dist[0, 2:]).all()
    grp.close()
    with pytest.raises(B.BvssError) as e:
        B.Group(V, off, devices=[], m=512, s=6, L=16)
    assert e.value.code == B.EINVAL
    with pytest.raises(B.BvssError) as e:
        B.Group(V, off, devices=[0, 99], m=512, s=6, L=16)
    assert e.value.code == B.EINVAL and "shard 1" in str(e.value)
