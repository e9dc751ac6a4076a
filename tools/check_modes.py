"""Developer check: default tensor-core refine vs exact SIMT refine on a medium
workload (many work items per CTA).  Not a test (needs minutes of GPU)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import synth
from paper_2412_03301_b200 import bvss as B
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
cfg = synth.get_config("cfg3", n=n, nq=nq, T=2000)
g = synth.generate(cfg, device="cuda")
res = {}
for terms in (0, 255):
    idx = B.Index(g["vectors"], g["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, seed=cfg.seed, refine_terms=terms, query_batch=int(os.environ.get("QB", "0")))
    ids, d = idx.search(g["queries"], g["q_offsets"], cfg.k, cfg.T)
    res[terms] = (ids.cpu().numpy(), d.cpu().numpy(), idx.stats())
    idx.close()
a, b = res[0], res[255]
same = (a[0] == b[0]).all(axis=1)
print("queries identical:", same.mean(), "max |dd|:", np.abs(a[1] - b[1]).max())
print("cand_rows tc:", a[2]["cand_rows"], "fixups:", a[2]["fixup_sets"])
bad = np.flatnonzero(~same)[:5]
for q in bad:
    print(q, a[0][q], b[0][q], a[1][q], b[1][q])
