"""Thin ctypes binding of libbvss (include/bvss.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels.  Host inputs
(numpy arrays) are passed as host pointers; torch CUDA tensors are passed as
device pointers with BVSS_DEVICE_PTRS, and the index is bound to torch's
current stream for the call so that ordering with surrounding torch work is
preserved.  There is no CPU fallback: if libbvss.so is missing the import of
this module raises, and if no sm_100 device is present the library returns
BVSS_EUNSUPPORTED, raised here as ``BvssError``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BVSS_LIB") or os.path.join(_HERE, "libbvss.so")  # BVSS_LIB: developer A/B of builds

OK, EINVAL, ENONFINITE, ENOMEM, ECUDA, EUNSUPPORTED, ESTATE, ENCCL = 0, -1, -2, -3, -4, -5, -6, -7
SKETCH_BINARY, SKETCH_COUNT_U8 = 0, 1
DEVICE_PTRS, VALIDATE_FINITE, KEEP_CODES = 0x1, 0x2, 0x4

# every symbol include/bvss.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "bvss_build_index", "bvss_search", "bvss_free_index", "bvss_last_error", "bvss_get_info", "bvss_get_stats",
    "bvss_set_stream", "bvss_device_count", "bvss_export_projection", "bvss_export_codes", "bvss_export_sketches",
    "bvss_query_sketch", "bvss_filter", "bvss_refine", "bvss_bruteforce", "bvss_index_begin", "bvss_index_append",
    "bvss_index_finish", "bvss_refine_error_bound", "bvss_dist_begin",
    "bvss_dist_hist", "bvss_dist_resolve", "bvss_dist_tie_counts", "bvss_dist_finish", "bvss_merge_topk",
    "bvss_dist_end", "bvss_group_build", "bvss_group_search", "bvss_group_shards", "bvss_group_shard",
    "bvss_free_group",
)


class BvssError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"bvss error {code}: {msg}")
        self.code = code


class Params(C.Structure):
    _fields_ = [("m", C.c_uint32), ("s", C.c_uint32), ("L", C.c_uint32), ("sketch", C.c_uint32),
                ("seed", C.c_uint64), ("projection", C.c_void_p), ("device", C.c_int32), ("flags", C.c_uint32),
                ("query_batch", C.c_uint32), ("refine_terms", C.c_uint32),
                ("select_mode", C.c_uint32), ("metric", C.c_uint32), ("score", C.c_uint32),
                ("gate_A", C.c_uint32), ("gate_M", C.c_uint32), ("filter", C.c_uint32)]

METRICS = {"hausdorff": 0, "meanmin": 1, "min": 2}  # bvss_metric (rerank distance)
SCORES = {"default": 0, "overlap": 1, "binarized": 2, "l1": 3}  # bvss_score_kind (filter score)
FILTERS = {"sketch": 0, "alg2": 1}  # candidate generation (bvss_params.filter)


class Info(C.Structure):
    _fields_ = [("n", C.c_int64), ("nvec", C.c_int64), ("d", C.c_int32), ("dpad", C.c_int32), ("m", C.c_uint32),
                ("s", C.c_uint32), ("L", C.c_uint32), ("sketch", C.c_uint32), ("device", C.c_int32),
                ("device_bytes", C.c_uint64), ("workspace_bytes", C.c_uint64)]


class Stats(C.Structure):
    _fields_ = [("ms_h2d", C.c_float), ("ms_encode", C.c_float), ("ms_scan", C.c_float), ("ms_select", C.c_float),
                ("ms_refine", C.c_float), ("ms_topk", C.c_float), ("ms_d2h", C.c_float), ("ms_total", C.c_float),
                ("scan_bytes", C.c_uint64), ("gather_bytes", C.c_uint64), ("cand_rows", C.c_uint64),
                ("fixup_sets", C.c_uint64), ("kernel_launches", C.c_int32), ("query_batch", C.c_int32),
                ("select_batches", C.c_uint64), ("select_fallbacks", C.c_uint64), ("scan_macs", C.c_uint64),
                ("dense_batches", C.c_uint64), ("dense_survivors", C.c_uint64), ("dense_emitted", C.c_uint64),
                ("dense_pairs", C.c_uint64), ("dense_flop", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2412_03301_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I64, I32, U32, VP = C.c_void_p, C.c_int64, C.c_int32, C.c_uint32, C.c_void_p
    sig = {
        "bvss_build_index": (C.c_int, [P, P, I64, I32, C.POINTER(Params), C.POINTER(VP)]),
        "bvss_search": (C.c_int, [VP, P, P, I64, I32, I32, P, P, U32]),
        "bvss_free_index": (None, [VP]),
        "bvss_last_error": (C.c_char_p, []),
        "bvss_get_info": (C.c_int, [VP, C.POINTER(Info)]),
        "bvss_get_stats": (C.c_int, [VP, C.POINTER(Stats)]),
        "bvss_set_stream": (C.c_int, [VP, VP]),
        "bvss_device_count": (C.c_int, []),
        "bvss_export_projection": (C.c_int, [VP, P]),
        "bvss_export_codes": (C.c_int, [VP, I64, I64, P]),
        "bvss_export_sketches": (C.c_int, [VP, I64, I64, P]),
        "bvss_query_sketch": (C.c_int, [VP, P, P, I64, P, P, U32]),
        "bvss_filter": (C.c_int, [VP, P, P, I64, I32, P, P, U32]),
        "bvss_refine": (C.c_int, [VP, P, P, I64, P, I32, I32, P, P, P, U32]),
        "bvss_bruteforce": (C.c_int, [VP, P, P, I64, I64, I32, P, P, U32]),
        "bvss_index_begin": (C.c_int, [I64, I64, I32, P, C.POINTER(VP)]),
        "bvss_index_append": (C.c_int, [VP, P, P, I64]),
        "bvss_index_finish": (C.c_int, [VP]),
        "bvss_refine_error_bound": (C.c_double, [VP, C.c_double]),
        "bvss_dist_begin": (C.c_int, [VP, P, P, I64, I32, I32, I64, U32, C.POINTER(VP), C.POINTER(I32)]),
        "bvss_dist_hist": (C.c_int, [VP, I32, P]),
        "bvss_dist_resolve": (C.c_int, [VP, I32, P]),
        "bvss_dist_tie_counts": (C.c_int, [VP, P]),
        "bvss_dist_finish": (C.c_int, [VP, P, I32, I32, P, P]),
        "bvss_merge_topk": (C.c_int, [VP, P, P, I32, I64, I32, P, P]),
        "bvss_dist_end": (None, [VP]),
        "bvss_group_build": (C.c_int, [P, P, I64, I32, C.POINTER(Params), I32, P, C.POINTER(VP)]),
        "bvss_group_search": (C.c_int, [VP, P, P, I64, I32, I32, P, P, U32]),
        "bvss_group_shards": (I32, [VP]),
        "bvss_group_shard": (C.c_int, [VP, I32, C.POINTER(VP), C.POINTER(I64)]),
        "bvss_free_group": (None, [VP]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def _check(code):
    if code != OK:
        raise BvssError(code, lib.bvss_last_error().decode(errors="replace"))


def device_count() -> int:
    return lib.bvss_device_count()


def _is_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


def _ptr(x):
    """(pointer, keepalive) for a numpy array or torch tensor (contiguous)."""
    if x is None:
        return None, None
    if hasattr(x, "data_ptr"):
        x = x.contiguous()
        return C.c_void_p(x.data_ptr()), x
    a = np.ascontiguousarray(x)
    return C.c_void_p(a.ctypes.data), a


class Index:
    """A device-resident BioVSS index over one database shard (one GPU)."""

    def __init__(self, vectors, offsets, *, m, s, L, sketch="binary", seed=0, device=0, keep_codes=False,
                 validate=False, projection=None, refine_terms=0, query_batch=0, select_mode=0,
                 metric="hausdorff", score="default", gate_A=0, gate_M=1, filter="sketch"):
        """gate_A / gate_M: BioVSS++ stage 1 (Alg 6 lines 1, 3-9; 0 = open); filter: "sketch" (Alg 6's sketch
        scan) or "alg2" (BioVSS Alg 2: Haus^H over the per-vector codes)."""
        dev = _is_cuda(vectors)
        if dev != _is_cuda(offsets):
            raise ValueError("vectors and offsets must both be host arrays or both CUDA tensors")
        if dev:
            import torch
            vectors = vectors.to(torch.float32).contiguous()
            offsets = offsets.to(torch.int64).contiguous()
            device = vectors.device.index
        else:
            vectors = np.ascontiguousarray(vectors, dtype=np.float32)
            offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        n = int(offsets.shape[0]) - 1
        d = int(vectors.shape[1])
        self.sketch_kind = "binary" if score == "binarized" else sketch  # BINARIZED: a binary index (R25)
        proj = None if projection is None else np.ascontiguousarray(projection, dtype=np.uint16)
        p = Params(m=m, s=s, L=L, sketch=SKETCH_BINARY if sketch == "binary" else SKETCH_COUNT_U8, seed=seed,
                   projection=(proj.ctypes.data if proj is not None else None), device=device,
                   flags=(DEVICE_PTRS if dev else 0) | (KEEP_CODES if keep_codes else 0) |
                   (VALIDATE_FINITE if validate else 0), query_batch=query_batch, refine_terms=refine_terms,
                   select_mode=select_mode, metric=METRICS[metric], score=SCORES[score], gate_A=gate_A,
                   gate_M=gate_M if gate_A else 0, filter=FILTERS[filter])
        self._h = C.c_void_p()
        vp, _k1 = _ptr(vectors)
        op, _k2 = _ptr(offsets)
        if dev:
            import torch
            torch.cuda.current_stream(device).synchronize()
        _check(lib.bvss_build_index(vp, op, n, d, C.byref(p), C.byref(self._h)))
        self.n, self.d, self.m, self.s, self.L, self.device = n, d, m, s, L, device

    @classmethod
    def from_chunks(cls, chunks, *, n_total, nvec_total, d, m, s, L, sketch="binary", seed=0, device=0,
                    keep_codes=False, projection=None, refine_terms=0, query_batch=0, select_mode=0,
                    metric="hausdorff", score="default"):
        """Streaming build (bvss_index_begin / append / finish): `chunks` yields host arrays
        (vectors [v][d] fp32, local_offsets [c+1] int64 starting at 0), sets in database order."""
        self = cls.__new__(cls)
        proj = None if projection is None else np.ascontiguousarray(projection, dtype=np.uint16)
        p = Params(m=m, s=s, L=L, sketch=SKETCH_BINARY if sketch == "binary" else SKETCH_COUNT_U8, seed=seed,
                   projection=(proj.ctypes.data if proj is not None else None), device=device,
                   flags=KEEP_CODES if keep_codes else 0, query_batch=query_batch, refine_terms=refine_terms,
                   select_mode=select_mode, metric=METRICS[metric], score=SCORES[score])
        self._h = C.c_void_p()
        _check(lib.bvss_index_begin(int(n_total), int(nvec_total), int(d), C.byref(p), C.byref(self._h)))
        try:
            for vec, off in chunks:
                vec = np.ascontiguousarray(vec, dtype=np.float32)
                off = np.ascontiguousarray(off, dtype=np.int64)
                _check(lib.bvss_index_append(self._h, C.c_void_p(vec.ctypes.data), C.c_void_p(off.ctypes.data),
                                             int(off.shape[0]) - 1))
            _check(lib.bvss_index_finish(self._h))
        except Exception:
            lib.bvss_free_index(self._h)
            self._h = C.c_void_p()
            raise
        self.sketch_kind = "binary" if score == "binarized" else sketch  # BINARIZED: a binary index (R25)
        self.n, self.d, self.m, self.s, self.L, self.device = int(n_total), int(d), m, s, L, device
        return self

    # ------------------------------------------------------------- helpers
    def _bind_stream(self, tensors):
        if any(_is_cuda(t) for t in tensors if t is not None):
            import torch
            st = torch.cuda.current_stream(self.device).cuda_stream
            # torch reports the legacy default stream as 0; the C ABI reads NULL as "the index's own
            # stream", so name the legacy stream explicitly (cudaStreamLegacy == 0x1) to stay ordered
            # with torch's work on it
            _check(lib.bvss_set_stream(self._h, C.c_void_p(st if st else 1)))
            return DEVICE_PTRS
        _check(lib.bvss_set_stream(self._h, None))
        return 0

    def _alloc(self, like_dev, shape, dtype):
        if like_dev:
            import torch
            tdt = {np.int64: torch.int64, np.float32: torch.float32, np.int32: torch.int32,
                   np.uint32: torch.int32, np.uint8: torch.uint8}[dtype]
            return torch.empty(shape, dtype=tdt, device=f"cuda:{self.device}")
        return np.empty(shape, dtype=dtype)

    def _queries(self, queries, q_offsets):
        dev = _is_cuda(queries)
        if dev != _is_cuda(q_offsets):
            raise ValueError("queries and q_offsets must both be host arrays or both CUDA tensors")
        if not dev:
            queries = np.ascontiguousarray(queries, dtype=np.float32)
            q_offsets = np.ascontiguousarray(q_offsets, dtype=np.int64)
        return queries, q_offsets, dev, int(q_offsets.shape[0]) - 1

    # ---------------------------------------------------------------- API
    def search(self, queries, q_offsets, k, T, validate=False):
        """bvss_search: returns (ids int64 [nq][k], dist fp32 [nq][k])."""
        queries, q_offsets, dev, nq = self._queries(queries, q_offsets)
        fl = self._bind_stream([queries]) | (VALIDATE_FINITE if validate else 0)
        ids = self._alloc(dev, (nq, k), np.int64)
        dist = self._alloc(dev, (nq, k), np.float32)
        qp, _a = _ptr(queries)
        op, _b = _ptr(q_offsets)
        _check(lib.bvss_search(self._h, qp, op, nq, k, T, _ptr(ids)[0], _ptr(dist)[0], fl))
        return ids, dist

    def filter(self, queries, q_offsets, T):
        """bvss_filter: candidates (ascending id, -1 padded) and their filter scores."""
        queries, q_offsets, dev, nq = self._queries(queries, q_offsets)
        fl = self._bind_stream([queries])
        cand = self._alloc(dev, (nq, T), np.int32)
        score = self._alloc(dev, (nq, T), np.int32)
        qp, _a = _ptr(queries)
        op, _b = _ptr(q_offsets)
        _check(lib.bvss_filter(self._h, qp, op, nq, T, _ptr(cand)[0], _ptr(score)[0], fl))
        return cand, score

    def refine(self, queries, q_offsets, cand, k, with_approx=True):
        """bvss_refine: top-k from given candidate lists; optionally the per-candidate tensor-core H^2."""
        queries, q_offsets, dev, nq = self._queries(queries, q_offsets)
        if not dev:
            cand = np.ascontiguousarray(cand, dtype=np.int32)
        T = int(cand.shape[1])
        fl = self._bind_stream([queries])
        ids = self._alloc(dev, (nq, k), np.int64)
        dist = self._alloc(dev, (nq, k), np.float32)
        approx = self._alloc(dev, (nq, T), np.float32) if with_approx else None
        qp, _a = _ptr(queries)
        op, _b = _ptr(q_offsets)
        cp, _c = _ptr(cand)
        _check(lib.bvss_refine(self._h, qp, op, nq, cp, T, k, _ptr(ids)[0], _ptr(dist)[0],
                               _ptr(approx)[0] if approx is not None else None, fl))
        return ids, dist, approx

    def bruteforce(self, queries, q_offsets, k, set_limit=0):
        """bvss_bruteforce (K8): exact top-k over sets [0, set_limit) (all when 0)."""
        queries, q_offsets, dev, nq = self._queries(queries, q_offsets)
        fl = self._bind_stream([queries])
        ids = self._alloc(dev, (nq, k), np.int64)
        dist = self._alloc(dev, (nq, k), np.float32)
        qp, _a = _ptr(queries)
        op, _b = _ptr(q_offsets)
        _check(lib.bvss_bruteforce(self._h, qp, op, nq, int(set_limit), k, _ptr(ids)[0], _ptr(dist)[0], fl))
        return ids, dist

    def query_sketch(self, queries, q_offsets, with_codes=False):
        queries, q_offsets, dev, nq = self._queries(queries, q_offsets)
        fl = self._bind_stream([queries])
        if self.sketch_kind == "binary":
            sk = self._alloc(dev, (nq, self.m // 32), np.uint32)
        else:
            sk = self._alloc(dev, (nq, self.m), np.uint8)
        nrows = int(q_offsets[-1])
        codes = self._alloc(dev, (nrows, self.m // 32), np.uint32) if with_codes else None
        qp, _a = _ptr(queries)
        op, _b = _ptr(q_offsets)
        _check(lib.bvss_query_sketch(self._h, qp, op, nq, _ptr(sk)[0], _ptr(codes)[0] if codes is not None else None,
                                     fl))
        return (sk, codes) if with_codes else sk

    def export_projection(self):
        out = np.empty((self.m, self.s), dtype=np.uint16)
        _check(lib.bvss_export_projection(self._h, C.c_void_p(out.ctypes.data)))
        return out

    def export_codes(self, first=0, count=None):
        info = self.info()
        count = info["nvec"] - first if count is None else count
        out = np.empty((count, self.m // 32), dtype=np.uint32)
        _check(lib.bvss_export_codes(self._h, first, count, C.c_void_p(out.ctypes.data)))
        return out

    def export_sketches(self, first=0, count=None):
        count = self.n - first if count is None else count
        if self.sketch_kind == "binary":
            out = np.empty((count, self.m // 32), dtype=np.uint32)
        else:
            out = np.empty((count, self.m), dtype=np.uint8)
        _check(lib.bvss_export_sketches(self._h, first, count, C.c_void_p(out.ctypes.data)))
        return out

    def error_bound(self, qnorm_max):
        return lib.bvss_refine_error_bound(self._h, float(qnorm_max))

    def info(self):
        i = Info()
        _check(lib.bvss_get_info(self._h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in i._fields_}

    def stats(self):
        s = Stats()
        _check(lib.bvss_get_stats(self._h, C.byref(s)))
        return s.as_dict()

    def close(self):
        if getattr(self, "_h", None):
            lib.bvss_free_index(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h


class Group:
    """A single-process multi-device index (bvss_group_*): the database sharded by contiguous set-id ranges
    over `devices` (CUDA ordinals; one may repeat), searched by the exact global-T protocol with in-process
    collectives.  Host arrays only."""

    def __init__(self, vectors, offsets, *, devices, m, s, L, sketch="binary", seed=0, refine_terms=0,
                 query_batch=0, select_mode=0, metric="hausdorff", score="default", gate_A=0, gate_M=1,
                 filter="sketch"):
        vectors = np.ascontiguousarray(vectors, dtype=np.float32)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        n, d = int(offsets.shape[0]) - 1, int(vectors.shape[1])
        devs = np.ascontiguousarray(devices, dtype=np.int32)
        p = Params(m=m, s=s, L=L, sketch=SKETCH_BINARY if sketch == "binary" else SKETCH_COUNT_U8, seed=seed,
                   projection=None, device=0, flags=0, query_batch=query_batch, refine_terms=refine_terms,
                   select_mode=select_mode, metric=METRICS[metric], score=SCORES[score], gate_A=gate_A,
                   gate_M=gate_M if gate_A else 0, filter=FILTERS[filter])
        self._h = C.c_void_p()
        _check(lib.bvss_group_build(C.c_void_p(vectors.ctypes.data), C.c_void_p(offsets.ctypes.data), n, d,
                                    C.byref(p), int(devs.shape[0]), C.c_void_p(devs.ctypes.data),
                                    C.byref(self._h)))
        self.n, self.d = n, d

    @property
    def shards(self):
        return lib.bvss_group_shards(self._h)

    def shard_stats(self, i):
        h, base = C.c_void_p(), C.c_int64()
        _check(lib.bvss_group_shard(self._h, i, C.byref(h), C.byref(base)))
        st = Stats()
        _check(lib.bvss_get_stats(h, C.byref(st)))
        return int(base.value), st.as_dict()

    def search(self, queries, q_offsets, k, T):
        queries = np.ascontiguousarray(queries, dtype=np.float32)
        q_offsets = np.ascontiguousarray(q_offsets, dtype=np.int64)
        nq = int(q_offsets.shape[0]) - 1
        ids = np.empty((nq, k), np.int64)
        dist = np.empty((nq, k), np.float32)
        _check(lib.bvss_group_search(self._h, C.c_void_p(queries.ctypes.data), C.c_void_p(q_offsets.ctypes.data),
                                     nq, k, T, C.c_void_p(ids.ctypes.data), C.c_void_p(dist.ctypes.data), 0))
        return ids, dist

    def close(self):
        if getattr(self, "_h", None):
            lib.bvss_free_group(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
