"""K1 encoder A/B (developer tool): the lane-per-vector kernel (BVSS_ENC_LANES=1) vs the warp-per-vector
kernel (default) -- build time of the same index and identical codes (export_codes).  The library reads the
switch per call, so both run in one process."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from gen import synth
from paper_2412_03301_b200 import bvss as B

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200000
cfg = synth.get_config(name, n=n, nq=10)
g = synth.generate(cfg, device="cuda")
nvec = int(g["offsets"][-1])
res = {}
for lanes in ("1", "0", "1", "0"):
    os.environ["BVSS_ENC_LANES"] = lanes
    torch.cuda.synchronize()
    t = time.time()
    idx = B.Index(g["vectors"], g["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed,
                  keep_codes=True)
    torch.cuda.synchronize()
    dt = time.time() - t
    codes = idx.export_codes(0, nvec)
    sk = idx.export_sketches()
    idx.close()
    if lanes in res:
        continue
    res[lanes] = (dt, codes, sk)
    print(f"{name} n={n} nvec={nvec} lanes={lanes}: build {dt * 1e3:.1f} ms", flush=True)
same = np.array_equal(res["1"][1], res["0"][1]) and np.array_equal(res["1"][2], res["0"][2])
print("codes identical:", same, flush=True)
if not same:
    bad = np.flatnonzero((res["1"][1] != res["0"][1]).any(1))
    print("differing vectors:", bad.size, bad[:10])
    sys.exit(1)
