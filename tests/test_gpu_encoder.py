"""The lane-per-vector K1 encoder (opt-in BVSS_ENC_LANES=1, csrc/encode.cu flyhash_lanes_kernel) against the
oracle's FlyHash + WTA (Def 7, Alg 1; readings R4 ties -> lower row, R8 summation order):
codes bit-exact modulo near-tie rows, exactly L ones, and identical to the default warp-per-vector kernel.
Covers s = 6 / 8 / 12 (the compiled widths), L = 1 and a compaction-heavy L, and ragged last tiles (vector counts are not multiples of 32)."""
import numpy as np
import pytest

from gen import synth
from oracle import bvss_oracle as O
from tests._common import codes_match_modulo_near_ties

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2412_03301_b200.bvss")

CASES = {
    "cfg1": ("cfg1", {}),                                   # m=512 s=6 L=16 d=64
    "cfg3_small": ("cfg3", dict(n=3001, nq=4)),             # m=1024 s=8 L=32 d=384
    "cfg4_small": ("cfg4", dict(n=1500, nq=4, d=128)),      # m=2048 s=12 L=64
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("L", [None, 1])
def test_lane_encoder_matches_oracle(case, L, monkeypatch):
    if B.device_count() < 1:
        pytest.fail("no sm_100 device visible to libbvss (the GPU tests must run on a B200)")
    name, ov = CASES[case]
    cfg = synth.get_config(name, **ov)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    V = data["vectors"]
    LL = cfg.L if L is None else L
    kw = dict(m=cfg.m, s=cfg.s, L=LL, sketch=cfg.sketch, seed=cfg.seed, keep_codes=True)
    monkeypatch.setenv("BVSS_ENC_LANES", "1")
    idx = B.Index(V, data["offsets"], **kw)
    lanes = idx.export_codes()
    idx.close()
    monkeypatch.setenv("BVSS_ENC_LANES", "0")
    idx = B.Index(V, data["offsets"], **kw)
    warp = idx.export_codes()
    idx.close()
    np.testing.assert_array_equal(lanes, warp)
    W = O.projection(cfg.seed, cfg.m, cfg.s, cfg.d)
    ora = O.encode(V, W, LL)
    ndiff = codes_match_modulo_near_ties(lanes, ora, V, W, LL, cfg.m)
    assert ndiff <= max(1, V.shape[0] // 10000)
    assert np.all(O.popcount_rows(lanes) == LL)
