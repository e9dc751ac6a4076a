"""Developer A/B of the dense kernel's runtime switches in ONE process (one index, env read per launch):
python tools/dense_env_ab.py N NQ 'ENV=a,ENV2=b' 'ENV=c' ...   (results must be identical for every setting)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from gen import synth
from paper_2412_03301_b200 import bvss as B

n, nq = int(sys.argv[1]), int(sys.argv[2])
settings = sys.argv[3:] or [""]
cfg = synth.get_config("cfg3", n=n, nq=nq)
g = synth.generate(cfg, device="cuda")
idx = B.Index(g["vectors"], g["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed)
qv, qo = g["queries"], g["q_offsets"]
base = None
for rep in range(3):
    for s in settings:
        env = dict(kv.split("=") for kv in s.split(";") if kv)
        for k_, v in env.items():
            os.environ[k_] = v
        ids, dd = idx.bruteforce(qv, qo, cfg.k)
        torch.cuda.synchronize()
        st = idx.stats()
        for k_ in env:
            del os.environ[k_]
        r = (ids.cpu().numpy(), dd.cpu().numpy())
        same = None
        if base is None:
            base = r
        else:
            same = bool(np.array_equal(r[0], base[0]) and np.array_equal(r[1], base[1]))
        print(f"rep {rep} [{s or 'default'}] dense {st['ms_refine']:.2f} ms ({st['dense_flop'] / st['ms_refine'] / 1e9:.1f} "
              f"TFLOP/s) survivors {st['dense_survivors']} emitted {st['dense_emitted']} same {same}", flush=True)
