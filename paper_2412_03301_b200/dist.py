"""Multi-GPU search: the database is sharded by contiguous set-id ranges, one
process per GPU (torch.distributed, NCCL over NVLink), queries replicated.

Exact global-T protocol.  Every rank
  1. encodes + sketches the query batch and scans its shard (local keys);
  2. per radix round r: local score histogram -> all-reduce(sum) -> resolve the
     digit of the GLOBAL threshold tau (C1);
  3. local count of keys tied at tau -> all-gather (C2); rank r takes all of its
     keys < tau plus max(0, min(eq_r, T - below - sum_{r'<r} eq_r')) of its
     lowest-id ties, so the union over ranks is exactly the single-GPU top-T
     (ids ascending inside a shard, shards ordered by id);
  4. refines its share and computes its local top-k;
  5. all-gather of the local top-k lists (C3) and the K7 merge kernel.
The candidate set and the returned top-k are therefore identical for any
number of ranks.  The collectives are plain torch.distributed calls; every
arithmetic step runs in libbvss kernels (LibShardOps).  The protocol is written
against a small ops interface so that its host logic is tested on CPU with the
gloo backend (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

HIST_BINS = 2048


class LibShardOps:
    """The per-rank phases, run by libbvss on this rank's GPU."""

    def __init__(self, index, id_base: int):
        from . import bvss
        self.B = bvss
        self.index = index
        self.id_base = int(id_base)
        self.ctx = None

    def begin(self, queries, q_offsets, k, T):
        B = self.B
        self.index._bind_stream([queries])
        ctx, rounds = C.c_void_p(), C.c_int32()
        B._check(B.lib.bvss_dist_begin(self.index.handle, C.c_void_p(queries.data_ptr()),
                                       C.c_void_p(q_offsets.data_ptr()), q_offsets.shape[0] - 1, k, T, self.id_base,
                                       B.DEVICE_PTRS, C.byref(ctx), C.byref(rounds)))
        self.ctx = ctx
        self.nq, self.k, self.dev = q_offsets.shape[0] - 1, k, queries.device
        return rounds.value

    def hist(self, r):
        h = torch.empty((self.nq, HIST_BINS), dtype=torch.int32, device=self.dev)
        self.B._check(self.B.lib.bvss_dist_hist(self.ctx, r, C.c_void_p(h.data_ptr())))
        return h

    def resolve(self, r, global_hist):
        self.B._check(self.B.lib.bvss_dist_resolve(self.ctx, r, C.c_void_p(global_hist.data_ptr())))

    def tie_counts(self):
        e = torch.empty(self.nq, dtype=torch.int64, device=self.dev)
        self.B._check(self.B.lib.bvss_dist_tie_counts(self.ctx, C.c_void_p(e.data_ptr())))
        return e

    def finish(self, all_eq, world, rank):
        ids = torch.empty((self.nq, self.k), dtype=torch.int64, device=self.dev)
        dd = torch.empty((self.nq, self.k), dtype=torch.float32, device=self.dev)
        self.B._check(self.B.lib.bvss_dist_finish(self.ctx, C.c_void_p(all_eq.data_ptr()), world, rank,
                                                  C.c_void_p(ids.data_ptr()), C.c_void_p(dd.data_ptr())))
        return ids, dd

    def merge(self, all_ids, all_d, world):
        out_i = torch.empty((self.nq, self.k), dtype=torch.int64, device=self.dev)
        out_d = torch.empty((self.nq, self.k), dtype=torch.float32, device=self.dev)
        self.B._check(self.B.lib.bvss_merge_topk(self.index.handle, C.c_void_p(all_ids.data_ptr()),
                                                 C.c_void_p(all_d.data_ptr()), world, self.nq, self.k,
                                                 C.c_void_p(out_i.data_ptr()), C.c_void_p(out_d.data_ptr())))
        return out_i, out_d

    def end(self):
        if self.ctx is not None:
            self.B.lib.bvss_dist_end(self.ctx)
            self.ctx = None


def sharded_search(ops, queries, q_offsets, k: int, T: int, n_total: int, group=None):
    """Run the exact global-T protocol for one query batch; every rank returns
    the same merged top-k (ids int64 [nq][k], dist fp32 [nq][k])."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    T_eff = min(int(T), int(n_total))
    rounds = ops.begin(queries, q_offsets, k, T_eff)
    try:
        for r in range(rounds):
            h = ops.hist(r)
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)      # C1
            ops.resolve(r, h)
        eq = ops.tie_counts()
        # outputs are allocated flat along dim 0 ([world * rows, ...]; gloo requires it) and viewed per rank
        all_eq = torch.empty((world * eq.shape[0],), dtype=eq.dtype, device=eq.device)
        dist.all_gather_into_tensor(all_eq, eq, group=group)           # C2
        all_eq = all_eq.view(world, -1)
        ids, dd = ops.finish(all_eq, world, rank)
        all_ids = torch.empty((world * ids.shape[0], ids.shape[1]), dtype=ids.dtype, device=ids.device)
        all_d = torch.empty((world * dd.shape[0], dd.shape[1]), dtype=dd.dtype, device=dd.device)
        dist.all_gather_into_tensor(all_ids, ids, group=group)         # C3
        dist.all_gather_into_tensor(all_d, dd, group=group)
        return ops.merge(all_ids.view(world, *ids.shape), all_d.view(world, *dd.shape), world)  # K7
    finally:
        ops.end()


def shard_range(n: int, world: int, rank: int):
    """Contiguous, balanced set-id range [lo, hi) of rank `rank`."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)
