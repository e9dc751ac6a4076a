"""Small end-to-end run for debugging on the GPU box (not a test)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from gen import synth
from paper_2412_03301_b200 import bvss as B
cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "cfg1")
if len(sys.argv) > 2:
    cfg = synth.get_config(cfg.name, n=int(sys.argv[2]), nq=int(sys.argv[3]), T=int(sys.argv[4]))
d = synth.to_numpy(synth.generate(cfg, device="cpu"))
idx = B.Index(d["vectors"], d["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed)
print("built", idx.info(), flush=True)
cand, score = idx.filter(d["queries"], d["q_offsets"], cfg.T)
print("filter ok", cand[0][:10], score[0][:10], flush=True)
ids, dist, approx = idx.refine(d["queries"], d["q_offsets"], cand, cfg.k)
print("refine ok", ids[0], dist[0], approx[0][:5], flush=True)
ids, dist = idx.search(d["queries"], d["q_offsets"], cfg.k, cfg.T)
print("search ok", ids[0], dist[0], idx.stats(), flush=True)
