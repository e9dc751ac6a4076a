"""Seeded synthetic vector-set workloads shaped like BASELINE.json configs[0..4].

This module is the ONLY code shared by the oracle side and the CUDA side: it
draws inputs (vectors, set offsets, query sets) and holds none of the method's
arithmetic (no projection, no WTA, no sketch, no distance).  It uses torch's
counter-based generators so the same call on the same device type is
reproducible; the parity tests pass one generated tensor to both sides.

Recipe (reading R10 for the gaps the configs leave open):
  * centroids: ``normalize(N(0, I_d))``;
  * set sizes: uniform on the config's inclusive range, or Zipf(1.5) clipped
    to [1, 100] (cfg4: P(1)=1/zeta(1.5)=0.383, mass of x>=100 lumped at 100);
  * each set draws ``c`` distinct centroids (c uniform on its range); each
    vector picks one of its set's centroids uniformly and is
    ``normalize(centroid + sigma * z)``, z ~ N(0, I_d)  ("noise_mode=per_coord",
    the literal reading of cfg1's N(0, 0.3^2 I); "total" divides sigma by
    sqrt(d) and is used only for the labelled sensitivity run);
  * queries: ``nq`` distinct source sets drawn uniformly; every source vector
    is perturbed by ``sigma_q * z`` (0.1) and renormalised; the source id is
    returned (it stays in the database, the expected rank-1 answer).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import torch

ZETA_1_5 = 2.612375348685488  # Riemann zeta(1.5)


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    size: tuple  # (lo, hi) inclusive, or ("zipf", s, hi)
    d: int
    n_centroids: int
    cents_per_set: tuple
    sigma: float
    m: int
    s: int
    L: int
    sketch: str  # "binary" | "count"
    nq: int
    k: int
    T: int
    sigma_q: float = 0.1
    T_sweep: tuple = field(default_factory=tuple)
    seed: int = 0


# BASELINE.json configs[0..4]; '*' values are the survey's readings (R7, R10).
CONFIGS = {
    "cfg1": Config("cfg1", 1_000, (2, 8), 64, 50, (1, 2), 0.3, 512, 6, 16, "binary", 10, 5, 50),
    "cfg2": Config("cfg2", 100_000, (1, 64), 384, 1000, (1, 3), 0.3, 1024, 8, 32, "count", 1000, 10, 2000),
    "cfg3": Config("cfg3", 1_000_000, (4, 32), 384, 5000, (1, 3), 0.3, 1024, 8, 32, "binary", 10_000, 10, 2000,
                   T_sweep=(500, 2000, 8000)),
    "cfg4": Config("cfg4", 1_000_000, ("zipf", 1.5, 100), 768, 5000, (1, 4), 0.3, 2048, 12, 64, "count",
                   10_000, 10, 4000),
    "cfg5": Config("cfg5", 4_000_000, (4, 28), 384, 5000, (1, 3), 0.3, 1024, 8, 32, "binary", 1000, 10, 2000),
}


def get_config(name: str, **overrides) -> Config:
    return replace(CONFIGS[name], **overrides)


def _zipf_clipped_cdf(s: float, hi: int) -> torch.Tensor:
    x = torch.arange(1, hi, dtype=torch.float64)
    if abs(s - 1.5) > 1e-12:
        raise ValueError("only Zipf(1.5) (cfg4) is supported")
    pmf = x.pow(-s) / ZETA_1_5
    cdf = torch.cumsum(pmf, 0)
    return torch.cat([cdf, torch.ones(1, dtype=torch.float64)])  # lump the tail at hi


def _sizes(cfg: Config, n: int, g: torch.Generator, device) -> torch.Tensor:
    if cfg.size[0] == "zipf":
        _, s, hi = cfg.size
        cdf = _zipf_clipped_cdf(s, hi).to(device)
        u = torch.rand(n, generator=g, device=device, dtype=torch.float64)
        return torch.searchsorted(cdf, u, right=True).clamp_(max=hi - 1) + 1
    lo, hi = cfg.size
    return torch.randint(lo, hi + 1, (n,), generator=g, device=device, dtype=torch.int64)


def _distinct_centroids(n: int, cmax: int, nc: int, g, device) -> torch.Tensor:
    ids = torch.randint(0, nc, (n, cmax), generator=g, device=device, dtype=torch.int64)
    for _ in range(64):
        dup = torch.zeros(n, dtype=torch.bool, device=device)
        for a in range(cmax):
            for b in range(a):
                dup |= ids[:, a] == ids[:, b]
        if not bool(dup.any()):
            return ids
        redraw = torch.randint(0, nc, (n, cmax), generator=g, device=device, dtype=torch.int64)
        ids = torch.where(dup[:, None], redraw, ids)
    raise RuntimeError("could not draw distinct centroids")


def _normalize(x: torch.Tensor) -> torch.Tensor:
    return x / x.norm(dim=1, keepdim=True).clamp_min(1e-30)


@torch.no_grad()
def generate(cfg: Config, device="cpu", noise_mode: str = "per_coord", chunk_sets: int = 65536,
             with_queries: bool = True) -> dict:
    """Draw one workload.  Returns a dict of torch tensors on ``device``:
    vectors fp32 [N][d], offsets int64 [n+1], queries fp32 [Nq][d],
    q_offsets int64 [nq+1], q_source int64 [nq]."""
    device = torch.device(device)
    g = torch.Generator(device=device)
    g.manual_seed(int(cfg.seed) * 1_000_003 + 17)
    d = cfg.d
    sig = cfg.sigma if noise_mode == "per_coord" else cfg.sigma / math.sqrt(d)
    sig_q = cfg.sigma_q if noise_mode == "per_coord" else cfg.sigma_q / math.sqrt(d)

    cents = _normalize(torch.randn(cfg.n_centroids, d, generator=g, device=device, dtype=torch.float32))
    sizes = _sizes(cfg, cfg.n, g, device)
    offsets = torch.zeros(cfg.n + 1, dtype=torch.int64, device=device)
    offsets[1:] = torch.cumsum(sizes, 0)
    N = int(offsets[-1])
    vectors = torch.empty(N, d, dtype=torch.float32, device=device)
    clo, chi = cfg.cents_per_set
    for s0 in range(0, cfg.n, chunk_sets):
        s1 = min(cfg.n, s0 + chunk_sets)
        ns = s1 - s0
        nc_set = torch.randint(clo, chi + 1, (ns,), generator=g, device=device, dtype=torch.int64)
        cids = _distinct_centroids(ns, chi, cfg.n_centroids, g, device)
        sz = sizes[s0:s1]
        set_of_vec = torch.repeat_interleave(torch.arange(ns, device=device), sz)
        pick = (torch.rand(set_of_vec.shape[0], generator=g, device=device, dtype=torch.float64)
                * nc_set[set_of_vec]).floor().to(torch.int64)
        pick = torch.minimum(pick, nc_set[set_of_vec] - 1)
        cen = cents[cids[set_of_vec, pick]]
        z = torch.randn(cen.shape, generator=g, device=device, dtype=torch.float32)
        vectors[int(offsets[s0]):int(offsets[s1])] = _normalize(cen + sig * z)
    out = {"vectors": vectors, "offsets": offsets, "config": cfg, "noise_mode": noise_mode}
    if with_queries:
        nq = min(cfg.nq, cfg.n)
        src = torch.randperm(cfg.n, generator=g, device=device)[:nq].to(torch.int64)
        qsz = sizes[src]
        q_off = torch.zeros(nq + 1, dtype=torch.int64, device=device)
        q_off[1:] = torch.cumsum(qsz, 0)
        rows = _gather_rows(offsets, src, qsz, device)
        base = vectors[rows]
        z = torch.randn(base.shape, generator=g, device=device, dtype=torch.float32)
        out.update(queries=_normalize(base + sig_q * z).contiguous(), q_offsets=q_off, q_source=src)
    return out


def _gather_rows(offsets, src, qsz, device):
    # vectorised concatenation of row ranges [offsets[i], offsets[i+1]) for i in src
    start = offsets[src]
    rep = torch.repeat_interleave(start, qsz)
    first = torch.zeros_like(qsz)
    first[1:] = torch.cumsum(qsz, 0)[:-1]
    within = torch.arange(int(qsz.sum()), device=device) - torch.repeat_interleave(first, qsz)
    return rep + within


def to_numpy(batch: dict) -> dict:
    """Host copies of a generated workload, for the oracle."""
    return {k: (v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in batch.items()}
