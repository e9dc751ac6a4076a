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


def _host_collectives(group) -> bool:
    """gloo moves host tensors; NCCL moves device tensors in place."""
    return dist.get_backend(group) == "gloo"


def _all_reduce_sum(t, group):
    if _host_collectives(group) and t.is_cuda:
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def _all_gather(t, world, group):
    """[world * rows, ...] concatenation of every rank's t (rank order)."""
    if _host_collectives(group) and t.is_cuda:
        h = t.cpu().contiguous()
        out = torch.empty((world * h.shape[0],) + tuple(h.shape[1:]), dtype=h.dtype)
        dist.all_gather_into_tensor(out, h, group=group)
        return out.to(t.device)
    out = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t, group=group)
    return out


def sharded_search(ops, queries, q_offsets, k: int, T: int, n_total: int, group=None):
    """Run the exact global-T protocol for one query batch; every rank returns
    the same merged top-k (ids int64 [nq][k], dist fp32 [nq][k])."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if int(T) < int(k):
        raise ValueError(f"T ({T}) < k ({k}) (reading R16)")
    T_eff = min(int(T), int(n_total))  # (may be < k when the database has fewer than k sets: padded results)
    rounds = ops.begin(queries, q_offsets, k, T_eff)
    try:
        for r in range(rounds):
            h = ops.hist(r)
            _all_reduce_sum(h, group)                                    # C1
            ops.resolve(r, h)
        eq = ops.tie_counts()
        all_eq = _all_gather(eq, world, group).view(world, -1)           # C2
        ids, dd = ops.finish(all_eq, world, rank)
        all_ids = _all_gather(ids, world, group)                         # C3
        all_d = _all_gather(dd, world, group)
        return ops.merge(all_ids.view(world, *ids.shape), all_d.view(world, *dd.shape), world)  # K7
    finally:
        ops.end()


def shard_range(n: int, world: int, rank: int):
    """Contiguous, balanced set-id range [lo, hi) of rank `rank`."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)
