"""Developer repro: small searches and a brute force with a ragged last chunk (run with BVSS_DEBUG_SYNC=1)."""
import sys; sys.path.insert(0, '.')
import numpy as np
from gen import synth
from paper_2412_03301_b200 import bvss as B
cfg = synth.get_config("cfg3", n=9000, nq=4)
data = synth.to_numpy(synth.generate(cfg, device="cpu"))
idx = B.Index(data["vectors"], data["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed)
for lim in (8192, 8500, 0):
    ids, d = idx.bruteforce(data["queries"], data["q_offsets"], cfg.k, set_limit=lim)
    print("ok", lim, ids[0][:3], flush=True)
