"""World-size-2/3 CPU tests (gloo backend) of the sharded search protocol in
paper_2412_03301_b200/dist.py.

The protocol's host logic -- the per-round all-reduce of score histograms (C1),
the all-gather of tie counts and the tie quota (C2), the all-gather of local
top-k lists (C3) and the merge -- runs exactly as on the GPU; only the per-rank
phases (`ops`) are replaced by a plain CPU implementation built on the oracle
(test infrastructure).  The merged result must equal the single-process oracle
search on the whole database for every world size, including budgets T whose
threshold ties straddle shard boundaries.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gen import synth
from oracle import bvss_oracle as O
from paper_2412_03301_b200 import dist as D

HIST_BITS = 11


class OracleShardOps:
    """The per-rank phases of the protocol on CPU (oracle scores, an
    independent numpy radix select, oracle Hausdorff refine)."""

    def __init__(self, oi: O.OracleIndex, id_base: int):
        self.oi = oi
        self.id_base = id_base

    def begin(self, queries, q_offsets, k, T):
        Qa = queries.numpy()
        qo = q_offsets.numpy()
        self.Q = [Qa[qo[i]:qo[i + 1]] for i in range(len(qo) - 1)]
        self.nq, self.k, self.teff = len(self.Q), k, T
        self.keys = np.stack([self.oi.scores(q).astype(np.int64) for q in self.Q])  # [nq][n_local]
        maxkey = self.oi.m if self.oi.kind == "binary" else self.oi.m * 255 * 255
        self.key_bits = int(maxkey).bit_length()
        self.rounds = -(-self.key_bits // HIST_BITS)
        self.prefix = np.zeros(self.nq, dtype=np.int64)
        self.below = np.zeros(self.nq, dtype=np.int64)
        self.digit = np.zeros(self.nq, dtype=np.int64)
        return self.rounds

    def _round(self, r):
        hi = self.key_bits - HIST_BITS * r
        shift = max(hi - HIST_BITS, 0)
        return hi, shift, hi - shift

    def hist(self, r):
        hi, shift, width = self._round(r)
        h = np.zeros((self.nq, D.HIST_BINS), dtype=np.int32)
        for q in range(self.nq):
            kq = self.keys[q]
            sel = (kq >> hi) == self.prefix[q]
            np.add.at(h[q], (kq[sel] >> shift) & ((1 << width) - 1), 1)
        self.last_local = h
        return torch.from_numpy(h)

    def resolve(self, r, global_hist):
        _, _, width = self._round(r)
        g = global_hist.numpy().astype(np.int64)
        for q in range(self.nq):
            cum = self.below[q] + np.cumsum(g[q])
            dg = int(np.searchsorted(cum, self.teff, side="left"))
            dg = min(dg, (1 << width) - 1)
            self.below[q] += int(g[q][:dg].sum())
            self.prefix[q] = (self.prefix[q] << width) | dg
            self.digit[q] = dg

    def tie_counts(self):
        return torch.tensor([int(self.last_local[q][self.digit[q]]) for q in range(self.nq)], dtype=torch.int64)

    def finish(self, all_eq, world, rank):
        ae = all_eq.numpy()
        ids = np.full((self.nq, self.k), -1, dtype=np.int64)
        dd = np.full((self.nq, self.k), np.inf, dtype=np.float32)
        for q in range(self.nq):
            left = self.teff - self.below[q] - int(ae[:rank, q].sum())
            quota = max(0, min(left, int(ae[rank, q])))
            kq, tau = self.keys[q], self.prefix[q]
            lt = np.flatnonzero(kq < tau)
            eq = np.flatnonzero(kq == tau)[:quota]
            cand = np.sort(np.concatenate([lt, eq]))
            if cand.size == 0:
                continue
            dist_ = O.refine(self.Q[q], cand, self.oi.vectors, self.oi.offsets)
            ri, rd = O.top_k(cand + self.id_base, dist_, self.k)
            ids[q], dd[q] = ri, rd
        return torch.from_numpy(ids), torch.from_numpy(dd)

    def merge(self, all_ids, all_d, world):
        ai = all_ids.numpy()
        ad = all_d.numpy().astype(np.float64)
        out_i = np.full((self.nq, self.k), -1, dtype=np.int64)
        out_d = np.full((self.nq, self.k), np.inf, dtype=np.float32)
        for q in range(self.nq):
            i = ai[:, q].reshape(-1)
            d_ = ad[:, q].reshape(-1)
            ok = i >= 0
            i, d_ = i[ok], d_[ok]
            order = np.lexsort((i, d_))[: self.k]
            out_i[q, : order.size] = i[order]
            out_d[q, : order.size] = d_[order]
        return torch.from_numpy(out_i), torch.from_numpy(out_d)

    def end(self):
        pass


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg_kw, T, k, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.get_config(**cfg_kw)
        data = synth.to_numpy(synth.generate(cfg, device="cpu"))
        lo, hi = D.shard_range(cfg.n, world, rank)
        off = data["offsets"]
        vec = data["vectors"][off[lo]:off[hi]]
        oi = O.OracleIndex(vec, off[lo:hi + 1] - off[lo], cfg.m, cfg.s, cfg.L, cfg.seed, sketch=cfg.sketch)
        ids, dd = D.sharded_search(OracleShardOps(oi, lo), torch.from_numpy(data["queries"]),
                                   torch.from_numpy(data["q_offsets"]), k, T, cfg.n)
        np.save(os.path.join(out_dir, f"ids{rank}.npy"), ids.numpy())
        np.save(os.path.join(out_dir, f"dist{rank}.npy"), dd.numpy())
    finally:
        dist.destroy_process_group()


def _single(cfg_kw, T, k):
    cfg = synth.get_config(**cfg_kw)
    data = synth.to_numpy(synth.generate(cfg, device="cpu"))
    oi = O.OracleIndex(data["vectors"], data["offsets"], cfg.m, cfg.s, cfg.L, cfg.seed, sketch=cfg.sketch)
    qo = data["q_offsets"]
    res = [oi.search(data["queries"][qo[i]:qo[i + 1]], k, min(T, cfg.n)) for i in range(cfg.nq)]
    return np.stack([r[0] for r in res]), np.stack([r[1] for r in res]).astype(np.float32)


@pytest.mark.parametrize("world,cfg_kw,T,k", [
    (2, dict(name="cfg1", n=300, nq=4), 50, 5),      # binary, 1 radix round
    (3, dict(name="cfg1", n=301, nq=3), 37, 5),      # uneven shards, odd T (ties straddle shards)
    (2, dict(name="cfg1", n=200, nq=3), 500, 5),     # T > n: exact brute force
    (2, dict(name="cfg2", n=120, nq=2, d=32), 40, 10),  # count sketch, 3 radix rounds
])
def test_sharded_protocol_matches_single_process(tmp_path, world, cfg_kw, T, k):
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, cfg_kw, T, k, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    ref_ids, ref_d = _single(cfg_kw, T, k)
    for r in range(world):
        ids = np.load(tmp_path / f"ids{r}.npy")
        dd = np.load(tmp_path / f"dist{r}.npy")
        np.testing.assert_array_equal(ids, ref_ids)
        np.testing.assert_array_equal(dd, ref_d)


@pytest.mark.parametrize("n,world", [(10, 3), (7, 7), (1000, 8), (5, 2)])
def test_shard_range_partitions(n, world):
    ranges = [D.shard_range(n, world, r) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    for (a, b), (c, _) in zip(ranges, ranges[1:]):
        assert b == c
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1
