"""A/B timing of developer switches inside ONE process (developer tool; not bench values).

The index is built once; each round runs every variant (a set of environment
variables the library reads at launch time) once, after a warm-up search, with
the L2 flushed before every search; prints the per-stage times of every run and
the median per variant, so box-to-box and process-order effects cancel.

    python tools/ab_env.py --var BVSS_REFINE_ATMEM=0 --var BVSS_REFINE_ATMEM=1 --rounds 3
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from gen import synth  # noqa: E402
from paper_2412_03301_b200 import bvss as B  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="cfg3")
    p.add_argument("--n", type=int, default=0)
    p.add_argument("--nq", type=int, default=0)
    p.add_argument("--var", action="append", default=[], help="'K=V[;K=V...]' (one variant; '' = defaults)")
    p.add_argument("--rounds", type=int, default=3)
    a = p.parse_args()
    over = {}
    if a.n:
        over["n"] = a.n
    if a.nq:
        over["nq"] = a.nq
    cfg = synth.get_config(a.config, **over)
    dev = torch.device("cuda:0")
    g = synth.generate(cfg, device=dev)
    idx = B.Index(g["vectors"], g["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed, device=0)
    del g["vectors"]
    torch.cuda.empty_cache()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    variants = a.var or [""]
    res = {v: [] for v in variants}
    base = dict(os.environ)
    ref = None
    for r in range(a.rounds + 1):
        for v in variants:
            os.environ.clear()
            os.environ.update(base)
            for kv in filter(None, v.split(";")):
                k, val = kv.split("=", 1)
                os.environ[k] = val
            flush.zero_()
            torch.cuda.synchronize()
            ids, _ = idx.search(g["queries"], g["q_offsets"], cfg.k, cfg.T)
            torch.cuda.synchronize()
            s = idx.stats()
            if ref is None:
                ref = ids.clone()
            same = bool(torch.equal(ids, ref))
            if r == 0:
                continue  # warm-up round
            res[v].append(s)
            print(f"round {r} [{v or 'default'}] refine {s['ms_refine']:.2f} scan {s['ms_scan']:.2f} "
                  f"topk {s['ms_topk']:.2f} total {s['ms_total']:.2f} ms  same-result {same}", flush=True)
    for v in variants:
        med = {k: statistics.median(x[k] for x in res[v]) for k in ("ms_refine", "ms_scan", "ms_topk", "ms_total")}
        print(f"median [{v or 'default'}] " + " ".join(f"{k} {val:.2f}" for k, val in med.items()))


if __name__ == "__main__":
    main()
