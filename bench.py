#!/usr/bin/env python
"""bench.py — BioVSS hot path on B200 (BASELINE.json metric):
"query sets/s at recall@10>=0.9 (1M sets, d=384); filter-scan HBM GB/s".

Workload (default): BASELINE.json configs[2] ("cfg3"): n = 1,000,000 sets of
uniform 4-32 unit vectors (d=384, ~18M vectors), 10,000 query sets, T = 2000,
k = 10, FlyHash m=1024 / s=8 / L=32, 1024-bit Bloom sketches.  Synthetic,
seeded, generated on the GPU (gen/synth.py).

A step = one bvss_search over the whole 10k-query batch against the resident
index (a-4 .. a-9: query encode + sketch, filter scan, top-T select, tensor-core
refine, exact top-k).  The index build (a-1 .. a-3) runs once before timing and
is reported separately under "build".  Inputs are device-resident when the
timed region starts; L2 is flushed (256 MB write) between timed steps and every
step is timed with CUDA events on the launching stream (the flush is outside the
events).  For N > 1 (torchrun, one process per GPU) the database is sharded by
contiguous set-id ranges and the exact global-T protocol runs over NCCL
(paper_2412_03301_b200/dist.py); value = 10k / max-over-ranks step time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "query sets/s at recall@10>=0.9 (1M sets, d=384); filter-scan HBM GB/s"
UNIT = "query sets/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--n", type=int, default=None, help="override the number of sets (quick runs only)")
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--T", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--terms", type=int, default=0, choices=[0, 1, 3, 255])
    ap.add_argument("--noise", default="per_coord", choices=["per_coord", "total"])
    ap.add_argument("--metric", default="hausdorff", choices=["hausdorff", "meanmin", "min"],
                    help="rerank distance (default: the paper's Hausdorff; MeanMin / Min are the §3.2 alternatives)")
    ap.add_argument("--recall-queries", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return {"hbm_gbs": j["hbm_gbs"], "bf16_tflops": j["bf16_tflops"], "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "src": "fallback"}


def workload_config(cfg, T, k):
    """The `config` both arms report (the same workload)."""
    return {"workload": (f"{cfg.name}: n={cfg.n} sets, d={cfg.d}, {cfg.nq} query sets, T={T}, k={k}, "
                         f"m={cfg.m}, s={cfg.s}, L={cfg.L}, {cfg.sketch} sketch"),
            "global_batch": cfg.nq}


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clock / throttle-reason samples every 100 ms.  The sampler is started before the warm-up
    (nvidia-smi's own start-up stalls the driver for milliseconds) and only the samples whose timestamp falls
    inside the timed region (`mark()` .. `stop()`) are reported."""
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None
        self.t0 = None
        self.t1 = None

    def mark(self):
        """Start of the timed region."""
        self.t0 = time.time()

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        self.t1 = time.time()
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)  # let the sample that covers the end of the timed region land
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        out = self.parse(self.path, self.t0, self.t1)
        os.unlink(self.path)
        return out

    @staticmethod
    def parse(path, t0, t1):
        """Median SM clock, max clock and the active throttle reasons of the samples in [t0, t1] (+-0.1 s);
        all samples if none carries a usable timestamp."""
        import datetime
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        with open(path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    ts = None
                rows.append((ts, parts[1:]))
        inside = [r for ts, r in rows if ts is not None and t0 is not None and t0 - 0.1 <= ts <= t1 + 0.1]
        for parts in (inside or [r for _, r in rows]):
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------- cpu baseline --
def oracle_sample(cfg, T, k, n_sample=10000, q_sample=3, seed_shift=0, metric="hausdorff"):
    """The oracle (as it stands, single-threaded numpy) on a bounded sample of
    the workload: a DB of n_sample sets drawn by the same generator recipe, and
    q_sample query sets.  Per query it times the query encode+sketch (a-4), the
    scan + top-T select over the sample (a-5, a-6), and the exact refine of T
    candidates + top-k (a-7, a-8); the scan/select time is scaled by n/n_sample
    (it is linear in n) and the refine time is the full-T cost.  Returns q/s
    for the FULL workload."""
    import numpy as np
    from gen import synth
    from oracle import bvss_oracle as O
    sc = synth.get_config(cfg.name, n=n_sample, nq=q_sample, seed=cfg.seed + seed_shift)
    data = synth.to_numpy(synth.generate(sc, device="cpu"))
    oi = O.OracleIndex(data["vectors"], data["offsets"], cfg.m, cfg.s, cfg.L, cfg.seed, sketch=cfg.sketch)
    Tr = min(T, n_sample)
    t_enc = t_scan = t_ref = 0.0
    for qi in range(q_sample):
        Q = data["queries"][data["q_offsets"][qi]:data["q_offsets"][qi + 1]]
        t0 = time.perf_counter()
        sq = oi.query_sketch(Q)
        t1 = time.perf_counter()
        scores = O.hamming_scores(sq, oi.sketches) if cfg.sketch == "binary" else O.count_l2_scores(sq, oi.sketches)
        cand = O.select_top_T(scores, Tr)
        t2 = time.perf_counter()
        dist = O.refine(Q, cand, oi.vectors, oi.offsets, metric)
        O.top_k(cand, dist, k)
        t3 = time.perf_counter()
        t_enc += t1 - t0
        t_scan += t2 - t1
        t_ref += (t3 - t2) * (T / Tr)
    per_q = (t_enc + t_scan * (cfg.n / n_sample) + t_ref) / q_sample
    sample = (f"oracle on {q_sample} query sets against a {n_sample}-set DB drawn by the {cfg.name} recipe; "
              f"scan+select time x{cfg.n / n_sample:g} (linear in n), exact refine of T={T} candidates timed as is; "
              f"index build not timed (as for the GPU)")
    return 1.0 / per_q, sample, per_q * q_sample


# ------------------------------------------------------------- our impl --
def main_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from gen import synth
    from paper_2412_03301_b200 import bvss as B
    from paper_2412_03301_b200 import dist as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("for --gpus > 1 launch with torchrun (one process per GPU)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    over = {}
    if args.n:
        over["n"] = args.n
    if args.nq:
        over["nq"] = args.nq
    if args.T:
        over["T"] = args.T
    if args.k:
        over["k"] = args.k
    cfg = synth.get_config(args.config, **over)
    T, k = cfg.T, cfg.k
    peaks = load_peaks()

    t0 = time.perf_counter()
    g = synth.generate(cfg, device=dev, noise_mode=args.noise)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    lo, hi = D.shard_range(cfg.n, world, rank)
    off_all = g["offsets"]
    vec = g["vectors"][int(off_all[lo]):int(off_all[hi])]
    off = (off_all[lo:hi + 1] - off_all[lo]).contiguous()
    qv, qo = g["queries"], g["q_offsets"]
    nvec_shard = int(off[-1])

    torch.cuda.synchronize()
    b0 = torch.cuda.Event(enable_timing=True)
    b1 = torch.cuda.Event(enable_timing=True)
    b0.record()
    idx = B.Index(vec, off, m=cfg.m, s=cfg.s, L=cfg.L, sketch=cfg.sketch, seed=cfg.seed, device=local,
                  refine_terms=args.terms, metric=args.metric)
    b1.record()
    torch.cuda.synchronize()
    build_ms = b0.elapsed_time(b1)
    if world == 1:
        del g["vectors"]
    del vec
    torch.cuda.empty_cache()

    def step():
        if world == 1:
            return idx.search(qv, qo, k, T)
        return D.sharded_search(D.LibShardOps(idx, lo), qv, qo, k, T, cfg.n)

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    clk = ClockSampler(local)
    clk.start()  # before the warm-up: nvidia-smi's start-up must not fall into the timed region
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.mark()
    st_sum, launches = {}, 0
    times = []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        th0 = time.perf_counter()
        out_ids, out_d = step()
        th1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        if os.environ.get("BVSS_TRACE"):
            print(f"[bench] step host {1000 * (th1 - th0):.1f} ms, events {e0.elapsed_time(e1):.1f} ms", file=sys.stderr)
        times.append(e0.elapsed_time(e1))
        s = idx.stats()
        launches += int(s["kernel_launches"]) + (0 if world == 1 else 1)
        for key in ("ms_encode", "ms_scan", "ms_select", "ms_refine", "ms_topk", "ms_h2d", "ms_total", "scan_bytes",
                    "gather_bytes", "cand_rows", "fixup_sets", "select_batches", "select_fallbacks", "scan_macs"):
            st_sum[key] = st_sum.get(key, 0) + s[key]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = clk.stop()
    total_ms = sum(times)
    if world > 1:
        tt = torch.tensor([total_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / args.steps
    value = cfg.nq / (ms_per_step / 1000.0)
    K = args.steps
    stages = {kk: st_sum[kk] / K for kk in ("ms_h2d", "ms_encode", "ms_scan", "ms_select", "ms_refine", "ms_topk", "ms_total")}

    # -------- roofline of the dominant kernel (algorithmic bytes / live event time)
    scan_bytes = st_sum["scan_bytes"] / K
    gather_bytes = st_sum["gather_bytes"] / K
    scan_gbs = scan_bytes / (stages["ms_scan"] * 1e-3) / 1e9 if stages["ms_scan"] > 0 else 0.0
    refine_gbs = gather_bytes / (stages["ms_refine"] * 1e-3) / 1e9 if stages["ms_refine"] > 0 else 0.0
    # K3 scan: an exact tensor-core contraction (FP4 kind::mxf4 for binary sketches, int8 kind::i8 for count
    # sketches): roofline = the measured bf16 dense peak x the nominal dense ratio of its dtype (fp4 4x, int8 2x)
    scan_flop = 2.0 * st_sum["scan_macs"] / K
    scan_tfs = scan_flop / (stages["ms_scan"] * 1e-3) / 1e12 if stages["ms_scan"] > 0 else 0.0
    scan_ratio = 4.0 if cfg.sketch == "binary" else 2.0
    scan_peak = peaks["bf16_tflops"] * scan_ratio
    roofs = {
        "scan": {"kernel": "scan_tc_kernel", "bound": "tensor", "achieved": round(scan_tfs, 1), "peak": round(scan_peak, 1),
                 "unit": "TFLOP/s", "frac": round(scan_tfs / scan_peak, 4), "ms": round(stages["ms_scan"], 3),
                 "flop_per_step": scan_flop, "db_operand_GBps": round(scan_gbs, 1),
                 "peak_src": f"{peaks['src']} bf16_tflops x {scan_ratio:g} (nominal dense "
                             f"{'fp4' if cfg.sketch == 'binary' else 'int8'}/bf16 ratio)"},
        "refine": {"kernel": "refine_tc_kernel", "bound": "hbm", "achieved": round(refine_gbs, 1),
                   "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(refine_gbs / peaks["hbm_gbs"], 4),
                   "ms": round(stages["ms_refine"], 3), "bytes_per_step": int(gather_bytes),
                   "peak_src": peaks["src"] + " (MEASURED_PEAKS.json hbm_gbs)"},
    }
    dom = max(roofs, key=lambda r: roofs[r]["ms"])
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(roofs[dom]["kernel"])
    roof = dict(roofs[dom], traffic=traffic)

    # -------- recall@10 against exact brute force (GPU, chunked exact refine over all ids), untimed
    recall = None
    if world == 1 and args.recall_queries > 0:
        recall = measure_recall(idx, qv, qo, out_ids, cfg, args.recall_queries, dev)

    # -------- e2e: the same metric through the C ABI with HOST buffers (pinned queries in, results out)
    e2e = None
    if world == 1 and not args.no_e2e:
        qh = torch.empty(qv.shape, dtype=torch.float32, pin_memory=True)
        qh.copy_(qv)
        qoh = qo.cpu().numpy()
        qhn = qh.numpy()
        idx.search(qhn, qoh, k, T)
        torch.cuda.synchronize()
        et = []
        for _ in range(max(1, min(args.steps, 3))):
            flush.zero_()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            ids_h, d_h = idx.search(qhn, qoh, k, T)
            et.append(time.perf_counter() - t1)
        h2d = qhn.nbytes + qoh.nbytes
        d2h = ids_h.nbytes + d_h.nbytes
        e2e = {"value": round(cfg.nq / statistics.mean(et), 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "timing": "host wall clock around bvss_search (host buffers)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        qps, sample, secs = oracle_sample(cfg, T, k, metric=args.metric)
        cpu = {"value": round(qps, 4), "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
               "cpu_seconds": round(secs, 1)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": ("e2m1 FP4 tensor-core scan (exact 0/1 products), " if cfg.sketch == "binary" else "u8 tensor-core scan, ") + "fp16 tensor-core Gram + exact fp32 fix-up (refine)",
            "data": f"synthetic (gen/synth.py {cfg.name} recipe, noise_mode={args.noise}), generated on GPU",
            "config": dict(workload_config(cfg, T, k), parallelism=f"db-shard{world}" if world > 1 else "single-gpu",
                           l2="flushed (256 MB write) before every timed step; DB 27.6 GB fp32 >> L2",
                           refine_terms=args.terms, query_batch=int(idx.stats()["query_batch"]),
                           **({} if args.metric == "hausdorff" else {"metric": args.metric})),
            "recall@10": recall["recall"] if recall else None,
            "recall": recall,
            "filter_scan_GBps": round(scan_gbs, 1),
            "filter_scan_TFLOPs": round(scan_tfs, 1),
            "stages_ms": {kk: round(v, 3) for kk, v in stages.items()},
            "roofline": roof,
            "roofline_all": roofs,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "build": {"ms": round(build_ms, 1), "vectors": nvec_shard,
                      "vectors_per_s": round(nvec_shard / (build_ms * 1e-3), 1), "gen_s": round(t_gen, 1),
                      "note": "index build (K1 encode + K9 split/norms + K2 sketch, incl. the D2D copy) per GPU"},
            "fixup_sets_per_step": st_sum["fixup_sets"] / K,
            "select": {"sampled_batches": st_sum["select_batches"], "fallbacks": st_sum["select_fallbacks"]},
        }
        print(json.dumps(line), flush=True)
    idx.close()
    if world > 1:
        dist.destroy_process_group()


def measure_recall(idx, qv, qo, out_ids, cfg, R, dev):
    """recall@k of the timed search's results on the first R queries,
    against exact brute force computed on the GPU by the exact refine over ALL
    set ids in chunks (T = n), merged on the host."""
    import numpy as np
    import torch
    R = min(R, cfg.nq)
    qo_h = qo[: R + 1].cpu().numpy()
    qsub = qv[: int(qo_h[-1])].contiguous()
    qo_d = qo[: R + 1].contiguous()
    chunk = 8192
    best_ids = np.full((R, 0), -1, dtype=np.int64)
    best_d = np.full((R, 0), np.inf, dtype=np.float32)
    t0 = time.perf_counter()
    for c0 in range(0, cfg.n, chunk):
        c1 = min(cfg.n, c0 + chunk)
        cand = torch.arange(c0, c1, dtype=torch.int32, device=dev).repeat(R, 1).contiguous()
        ids, dd, _ = idx.refine(qsub, qo_d, cand, cfg.k, with_approx=False)
        best_ids = np.concatenate([best_ids, ids.cpu().numpy()], axis=1)
        best_d = np.concatenate([best_d, dd.cpu().numpy()], axis=1)
        order = np.lexsort((best_ids, best_d), axis=1)[:, : cfg.k]
        best_ids = np.take_along_axis(best_ids, order, 1)
        best_d = np.take_along_axis(best_d, order, 1)
    got = out_ids[:R].cpu().numpy()
    rec = [len(set(got[i].tolist()) & set(best_ids[i].tolist())) / cfg.k for i in range(R)]
    return {"recall": round(float(np.mean(rec)), 4), "queries": R, "k": cfg.k,
            "rank1_hit": round(float(np.mean([got[i][0] == best_ids[i][0] for i in range(R)])), 4),
            "ground_truth": "exact Hausdorff over all n sets on GPU (bvss_refine, T=n in chunks)",
            "seconds": round(time.perf_counter() - t0, 1)}


def main_reference(args):
    """Reference arm: the CPU oracle as it stands (there is no reference
    implementation to install: /root/reference holds only the paper)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from gen import synth
    over = {}
    if args.n:
        over["n"] = args.n
    if args.T:
        over["T"] = args.T
    cfg = synth.get_config(args.config, **over)
    for w in range(args.warmup):
        oracle_sample(cfg, cfg.T, cfg.k, n_sample=2000, q_sample=1, seed_shift=100 + w, metric=args.metric)
    vals, secs = [], 0.0
    sample = ""
    for s in range(args.steps):
        qps, sample, sec = oracle_sample(cfg, cfg.T, cfg.k, n_sample=5000, q_sample=1, seed_shift=s,
                                         metric=args.metric)
        vals.append(1.0 / qps)
        secs += sec
    ms_per_step = statistics.mean(vals) * 1000.0
    value = 1.0 / statistics.mean(vals)
    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64 (oracle)", "impl": "reference",
            "data": f"synthetic ({cfg.name} recipe)",
            "config": dict(workload_config(cfg, cfg.T, cfg.k), parallelism="cpu-oracle",
                           **({} if args.metric == "hausdorff" else {"metric": args.metric})),
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        main_reference(a)
    else:
        main_ours(a)
