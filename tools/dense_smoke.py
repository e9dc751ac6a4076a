"""Dense-path bring-up (developer tool): one small brute force through the dense kernel vs bvss_refine."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from gen import synth
from paper_2412_03301_b200 import bvss as B

cfg = synth.get_config("cfg3", n=int(sys.argv[1]) if len(sys.argv) > 1 else 3000, nq=int(sys.argv[2]) if len(sys.argv) > 2 else 50)
data = synth.to_numpy(synth.generate(cfg, device="cpu"))
idx = B.Index(data["vectors"], data["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed)
for rep in range(2):
    t = time.time()
    ids, dist = idx.bruteforce(data["queries"], data["q_offsets"], cfg.k)
    st = idx.stats()
    print("dense bruteforce %.3f s: dense %.2f ms (%.1f TFLOP/s), topk %.2f ms, survivors %d emitted %d" % (
        time.time() - t, st["ms_refine"], st["dense_flop"] / st["ms_refine"] / 1e9, st["ms_topk"],
        st["dense_survivors"], st["dense_emitted"]), flush=True)
if cfg.n > 20000:
    sys.exit(0)
cand = np.tile(np.arange(cfg.n, dtype=np.int32), (cfg.nq, 1))
r_ids, r_d, _ = idx.refine(data["queries"], data["q_offsets"], cand, cfg.k)
print("ids equal", np.array_equal(ids, r_ids), "dist equal", np.array_equal(dist, r_d))
bad = np.flatnonzero((ids != r_ids).any(1))
print("bad queries", bad[:10], len(bad))
if len(bad):
    q = bad[0]
    print(ids[q], r_ids[q]); print(dist[q], r_d[q])
