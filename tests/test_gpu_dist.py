"""The sharded search through the library's real phases (bvss_dist_* + K7 merge,
paper_2412_03301_b200/dist.py LibShardOps) on the GPU: two processes, each
holding one contiguous shard of the database as its own index on cuda:0, the
collectives over gloo (CUDA tensors staged through the host; only one GPU is
available here, and the protocol has no kernel that waits on another rank).
The merged top-k must equal the single-index search exactly (same kernels on
every (query, set) pair; global top-T by the exact tie protocol)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg_kw, out_dir, backend="gloo"):
    import torch
    import torch.distributed as dist
    from gen import synth
    from paper_2412_03301_b200 import bvss as B
    from paper_2412_03301_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if backend == "nccl":
        torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cfg = synth.get_config(**cfg_kw)
        g = synth.generate(cfg, device="cuda")
        lo, hi = D.shard_range(cfg.n, world, rank)
        off = g["offsets"]
        vec = g["vectors"][int(off[lo]):int(off[hi])].contiguous()
        idx = B.Index(vec, (off[lo:hi + 1] - off[lo]).contiguous(), m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch,
                      seed=cfg.seed)
        ids, dd = D.sharded_search(D.LibShardOps(idx, lo), g["queries"], g["q_offsets"], cfg.k, cfg.T, cfg.n)
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, f"ids{rank}.npy"), ids.cpu().numpy())
        np.save(os.path.join(out_dir, f"dist{rank}.npy"), dd.cpu().numpy())
        idx.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg_kw", [(2, dict(name="cfg3", n=6001, nq=9, T=300)),
                                          (3, dict(name="cfg2", n=3001, nq=5, T=120, d=64)),
                                          (2, dict(name="cfg1", n=500, nq=6, T=600))])
def test_sharded_search_equals_single_index(tmp_path, world, cfg_kw):
    import torch
    import torch.multiprocessing as mp
    from gen import synth
    from paper_2412_03301_b200 import bvss as B
    if B.device_count() < 1:
        pytest.fail("no sm_100 device visible to libbvss")
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, cfg_kw, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    cfg = synth.get_config(**cfg_kw)
    g = synth.generate(cfg, device="cuda")
    idx = B.Index(g["vectors"], g["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed,
                  select_mode=1)
    ref_ids, ref_d = idx.search(g["queries"], g["q_offsets"], cfg.k, cfg.T)
    idx.close()
    ref_ids, ref_d = ref_ids.cpu().numpy(), ref_d.cpu().numpy()
    for r in range(world):
        ids = np.load(tmp_path / f"ids{r}.npy")
        dd = np.load(tmp_path / f"dist{r}.npy")
        np.testing.assert_array_equal(ids, ref_ids)
        np.testing.assert_array_equal(dd, ref_d)


def test_sharded_search_matches_oracle(tmp_path):
    """The merged sharded result against the oracle pipeline (not only against the single-index GPU path):
    world size 2, a query subset checked by the tie-tolerant rule (Def 4, Alg 6)."""
    import torch.multiprocessing as mp
    from gen import synth
    from oracle import bvss_oracle as O
    from paper_2412_03301_b200 import bvss as B
    from tests._common import check_topk
    if B.device_count() < 1:
        pytest.fail("no sm_100 device visible to libbvss")
    cfg_kw = dict(name="cfg3", n=4001, nq=6, T=250)
    world = 2
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, cfg_kw, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    cfg = synth.get_config(**cfg_kw)
    h = synth.to_numpy(synth.generate(cfg, device="cuda"))  # the workers' exact data (CUDA generator)
    oi = O.OracleIndex(h["vectors"], h["offsets"], cfg.m, cfg.s, cfg.L, cfg.seed, sketch=cfg.sketch)
    ids = np.load(tmp_path / "ids0.npy")
    dd = np.load(tmp_path / "dist0.npy")
    V, off = h["vectors"], h["offsets"]
    for qi in range(cfg.nq):
        Q = h["queries"][h["q_offsets"][qi]:h["q_offsets"][qi + 1]]
        r_ids, r_d = oi.search(Q, cfg.k, cfg.T)
        check_topk(ids[qi], dd[qi], r_ids, r_d, lambda i: O.hausdorff(Q, V[off[i]:off[i + 1]]))


@pytest.mark.parametrize("cfg_kw", [dict(name="cfg3", n=6001, nq=9, T=300), dict(name="cfg3", n=5003, nq=7, T=4000)])
def test_sharded_search_over_nccl_one_rank(tmp_path, cfg_kw):
    """The collectives on CUDA tensors through NCCL (dist._host_collectives is false for nccl): one rank, the
    only NCCL world one GPU allows (NCCL rejects two ranks on one device).  C1 all-reduce, C2/C3 all-gathers run
    as NCCL kernels on the device buffers; the result must equal the single-index search exactly, both at a
    small T (sorted top-T) and at T close to n (bitmap + dense refine in bvss_dist_finish)."""
    import torch.multiprocessing as mp
    from gen import synth
    from paper_2412_03301_b200 import bvss as B
    if B.device_count() < 1:
        pytest.fail("no sm_100 device visible to libbvss")
    port = _free_port()
    mp.start_processes(_worker, args=(1, port, cfg_kw, str(tmp_path), "nccl"), nprocs=1, join=True,
                       start_method="spawn")
    cfg = synth.get_config(**cfg_kw)
    g = synth.generate(cfg, device="cuda")
    idx = B.Index(g["vectors"], g["offsets"], m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed,
                  select_mode=1)
    ref_ids, ref_d = idx.search(g["queries"], g["q_offsets"], cfg.k, cfg.T)
    idx.close()
    np.testing.assert_array_equal(np.load(tmp_path / "ids0.npy"), ref_ids.cpu().numpy())
    np.testing.assert_array_equal(np.load(tmp_path / "dist0.npy"), ref_d.cpu().numpy())
