"""Dense-path debugging (developer tool): the oversize-set workload of tests/test_gpu_scale.py."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import bvss_oracle as O
from paper_2412_03301_b200 import bvss as B
from tests._common import offsets_from_sizes
from tests.test_gpu_scale import _oversize_db

for big in (300, 200):
    rng = np.random.default_rng(5)
    Q, X, off = _oversize_db(rng, 64)
    if big != 300:  # rebuild with smaller big sets
        sizes = np.diff(off)
        keep = []
        for i in range(len(sizes)):
            s = X[off[i]:off[i + 1]]
            keep.append(s[:big] if s.shape[0] > big else s)
        X = np.concatenate(keep).astype(np.float32)
        off = offsets_from_sizes([s.shape[0] for s in keep])
    n = off.shape[0] - 1
    qo = np.array([0, Q.shape[0]], dtype=np.int64)
    idx = B.Index(X, off, m=256, s=4, L=16, seed=2)
    k = 10
    ids, dist = idx.bruteforce(Q, qo, k)
    st = idx.stats()
    cand = np.arange(n, dtype=np.int32)[None, :]
    r_ids, r_d, ap = idx.refine(Q, qo, cand, k)
    h = O.refine(Q, np.arange(n), X, off)
    o_ids, o_d = O.top_k(np.arange(n), h, k)
    print("big", big, "dense_batches", st["dense_batches"], "emitted", st["dense_emitted"], "surv", st["dense_survivors"])
    print(" dense ", ids[0].tolist()); print(" qmajor", r_ids[0].tolist()); print(" oracle", o_ids.tolist())
    print(" dense d", np.round(dist[0], 4).tolist()); print(" oracle d", np.round(o_d, 4).tolist())
    print(" sizes of oracle ids", [int(off[i + 1] - off[i]) for i in o_ids])
