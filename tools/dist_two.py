"""Developer check: the sharded protocol with world = 2 (gloo, one GPU), phase by phase."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist, torch.multiprocessing as mp

def work(rank, world):
    from gen import synth
    from paper_2412_03301_b200 import bvss as B
    from paper_2412_03301_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = "29544"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg = synth.get_config("cfg3", n=6001, nq=9, T=300)
    g = synth.generate(cfg, device="cuda")
    lo, hi = D.shard_range(cfg.n, world, rank)
    off = g["offsets"]
    idx = B.Index(g["vectors"][int(off[lo]):int(off[hi])].contiguous(), (off[lo:hi + 1] - off[lo]).contiguous(),
                  m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed)
    ops = D.LibShardOps(idx, lo)
    rounds = ops.begin(g["queries"], g["q_offsets"], cfg.k, cfg.T)
    for r in range(rounds):
        h = ops.hist(r)
        torch.cuda.synchronize()
        print(rank, "local hist sum", h.sum(1).tolist(), flush=True)
        D._all_reduce_sum(h, None)
        torch.cuda.synchronize()
        print(rank, "global hist sum", h.sum(1).tolist(), flush=True)
        ops.resolve(r, h)
    eq = ops.tie_counts()
    all_eq = D._all_gather(eq, world, None).view(world, -1)
    torch.cuda.synchronize()
    print(rank, "all_eq", all_eq.tolist(), flush=True)
    ids, dd = ops.finish(all_eq, world, rank)
    torch.cuda.synchronize()
    print(rank, "local ids q0", ids[0].tolist(), dd[0].tolist()[:3], flush=True)
    all_ids = D._all_gather(ids, world, None)
    all_d = D._all_gather(dd, world, None)
    torch.cuda.synchronize()
    print(rank, "gathered", all_ids.shape, all_ids[:, :3].tolist(), flush=True)
    mi, md = ops.merge(all_ids.view(world, *ids.shape), all_d.view(world, *dd.shape), world)
    torch.cuda.synchronize()
    print(rank, "merged", mi[:, 0].tolist(), flush=True)
    si, sd = D.sharded_search(D.LibShardOps(idx, lo), g["queries"], g["q_offsets"], cfg.k, cfg.T, cfg.n)
    torch.cuda.synchronize()
    print(rank, "sharded_search", si[:, 0].tolist(), flush=True)
    ops.end()
    dist.destroy_process_group()

if __name__ == "__main__":
    mp.start_processes(work, args=(2,), nprocs=2, join=True, start_method="spawn")
