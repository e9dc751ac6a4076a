"""K1 encoder A/B across library builds (developer tool): index build time of the same cfg3 database with each
libbvss.so given on the command line (BVSS_LIB per subprocess), and identical codes."""
import os, subprocess, sys, json
libs = sys.argv[1:]
code = r'''
import os, sys, time, json, numpy as np, torch
sys.path.insert(0, ".")
from gen import synth
from paper_2412_03301_b200 import bvss as B
cfg = synth.get_config("cfg3", n=400000, nq=10)
g = synth.generate(cfg, device="cuda")
nvec = int(g["offsets"][-1])
ts = []
for rep in range(3):
    torch.cuda.synchronize(); t = time.time()
    idx = B.Index(g["vectors"], g["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed, keep_codes=True)
    torch.cuda.synchronize(); ts.append(time.time() - t)
    if rep < 2: idx.close()
codes = idx.export_codes(0, nvec)
np.save(sys.argv[1], codes)
print(json.dumps({"nvec": nvec, "build_ms": [round(x * 1e3, 1) for x in ts]}))
'''
res = {}
for i, lib in enumerate(libs):
    env = dict(os.environ, BVSS_LIB=lib if lib != "new" else "")
    out = subprocess.run([sys.executable, "-c", code, f"/tmp/codes{i}.npy"], env=env, capture_output=True, text=True)
    print(lib, out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-2000:], flush=True)
import numpy as np
c0 = np.load("/tmp/codes0.npy")
for i in range(1, len(libs)):
    print(libs[i], "codes identical to", libs[0], np.array_equal(c0, np.load(f"/tmp/codes{i}.npy")))
