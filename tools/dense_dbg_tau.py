"""Developer: which tau source breaks the dense brute force on a small case (BVSS_DENSE_DEBUG 8..11, 0)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import synth
from oracle import bvss_oracle as O
import paper_2412_03301_b200.bvss as B

cfg = synth.get_config("cfg3", n=int(os.environ.get("N", 5003)), nq=40)
data = synth.to_numpy(synth.generate(cfg, device="cpu"))
limit = int(os.environ.get("LIMIT", 3001))
V, off = data["vectors"], data["offsets"]
H = []
for qi in range(cfg.nq):
    Q = data["queries"][data["q_offsets"][qi]:data["q_offsets"][qi + 1]]
    H.append(O.refine(Q, np.arange(limit), V, off))
for dbg in os.environ.get("DBGS", "8 9 10 11 0").split():
    os.environ["BVSS_DENSE_DEBUG"] = dbg
    idx = B.Index(V, off, m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed)
    ids, dist = idx.bruteforce(data["queries"], data["q_offsets"], cfg.k, set_limit=limit)
    st = idx.stats()
    bad = 0
    for qi in range(cfg.nq):
        h = H[qi]
        kth = np.sort(h)[cfg.k - 1]
        got = ids[qi][ids[qi] >= 0]
        if np.any(h[got] > kth * (1 + 1e-5)):
            bad += 1
    print(f"debug {dbg}: dense_batches {st['dense_batches']} survivors {st['dense_survivors']} "
          f"emitted {st['dense_emitted']} bad queries {bad}/{cfg.nq}", flush=True)
    idx.close()
