"""TEST INFRASTRUCTURE ONLY: Python bindings of the CPU oracle.

  Oracle  -- oracle/_build/libgenie_oracle.so, the plain-C restatement of the
             reference algorithm (oracle/genie_oracle.c)
  RefLib  -- oracle/_ref/libmcx_ref.so, the unmodified reference headers
             (/root/reference/proj/include) behind a C shim (oracle/ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module, and only as the checker or the reported
CPU baseline.  The product (paper_1603_08390_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libgenie_oracle.so"
REF_SO = HERE / "_ref" / "libmcx_ref.so"

u16p = C.POINTER(C.c_uint16)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def threads() -> int:
    return max(1, os.cpu_count() or 1)


class OracleResult:
    def __init__(self, qid, ids, counts, length, threshold, bound=None, postings=None):
        self.qid, self.ids, self.counts, self.length, self.threshold = qid, ids, counts, length, threshold
        self.bound, self.postings = bound, postings

    def row(self, q):
        n = int(self.length[q])
        return list(zip(self.ids[q, :n].tolist(), self.counts[q, :n].tolist()))


class Oracle:
    """The C restatement."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"oracle not built: {path} (make -C oracle)")
        L = C.CDLL(str(path))
        L.or_mix64.restype, L.or_mix64.argtypes = C.c_uint64, [C.c_uint64]
        L.or_index_create.restype = vp
        L.or_index_create.argtypes = [C.c_uint32, C.c_uint64, u64p, u64p, u32p]
        L.or_index_free.argtypes = [vp]
        L.or_max_multiplicity.restype, L.or_max_multiplicity.argtypes = C.c_uint32, [vp, C.c_uint32]
        L.or_max_count_bound.restype = C.c_uint64
        L.or_max_count_bound.argtypes = [vp, C.c_uint32, u16p, u32p, u32p]
        L.or_width_for.restype, L.or_width_for.argtypes = C.c_uint32, [C.c_uint32]
        L.or_execute.restype = C.c_int
        L.or_execute.argtypes = [vp, C.c_uint32, u32p, u32p, u64p, u16p, u32p, u32p, C.c_uint32, u32p, u32p, u32p,
                                 u32p, u64p, u64p, C.c_uint32, u32p]
        L.or_cpq_stream.restype = C.c_int
        L.or_cpq_stream.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, u32p, C.c_uint32, u32p, u32p,
                                    u32p, u32p, u32p, u32p]
        L.or_merge_topk.restype = C.c_int
        L.or_merge_topk.argtypes = [C.c_uint32, u64p, u32p, u32p, C.c_uint32, C.c_uint32, u32p, u32p, u32p, u32p]
        L.or_hash_results.restype = C.c_uint64
        L.or_hash_results.argtypes = [C.c_uint32, u32p, u32p, u32p, C.c_uint32, u32p, u32p]
        L.or_lsh_params.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_double, C.c_double, f64p, f64p,
                                    u64p, u64p]
        L.or_lsh_encode.argtypes = [C.c_int, C.c_uint32, C.c_uint32, f64p, f64p, C.c_double, C.c_uint32, C.c_int64,
                                    C.c_int, u64p, u64p, C.c_uint32, f32p, u64p, u64p, C.c_uint64, C.c_uint32, u32p]
        L.or_kernel_width.restype = C.c_double
        L.or_kernel_width.argtypes = [f32p, C.c_uint64, C.c_uint32, C.c_uint64]
        self.L = L

    def mix64(self, x: int) -> int:
        return int(self.L.or_mix64(x))

    def width_for(self, b: int) -> int:
        return int(self.L.or_width_for(b))

    def index(self, csr) -> "OracleIndex":
        return OracleIndex(self, csr)

    def cpq_stream(self, n, max_count, k, stream):
        s = np.ascontiguousarray(stream, np.uint32)
        cap = max(1, min(k, n) + k)
        ids, counts = np.zeros(cap, np.uint32), np.zeros(cap, np.uint32)
        ln, thr, at = C.c_uint32(), C.c_uint32(), C.c_uint32()
        za = np.zeros(max_count + 1, np.uint32)
        rc = self.L.or_cpq_stream(n, max_count, k, s.shape[0], _p(s, C.c_uint32), cap, _p(ids, C.c_uint32),
                                  _p(counts, C.c_uint32), C.byref(ln), C.byref(thr), C.byref(at), _p(za, C.c_uint32))
        return rc, list(zip(ids[: ln.value].tolist(), counts[: ln.value].tolist())), thr.value, at.value, za

    def merge_topk(self, lists, k):
        off = np.zeros(len(lists) + 1, np.uint64)
        ids, counts = [], []
        for i, l in enumerate(lists):
            off[i + 1] = off[i] + len(l)
            ids += [e[0] for e in l]
            counts += [e[1] for e in l]
        ids_a, counts_a = np.array(ids + [0], np.uint32), np.array(counts + [0], np.uint32)
        cap = max(1, int(off[-1]))
        oi, oc = np.zeros(cap, np.uint32), np.zeros(cap, np.uint32)
        ln, thr = C.c_uint32(), C.c_uint32()
        rc = self.L.or_merge_topk(len(lists), _p(off, C.c_uint64), _p(ids_a, C.c_uint32), _p(counts_a, C.c_uint32),
                                  k, cap, _p(oi, C.c_uint32), _p(oc, C.c_uint32), C.byref(ln), C.byref(thr))
        return rc, list(zip(oi[: ln.value].tolist(), oc[: ln.value].tolist())), thr.value

    def hash_results(self, qid, threshold, length, ids, counts) -> int:
        Q = len(qid)
        stride = ids.shape[1] if Q else 1
        a = [np.ascontiguousarray(x, np.uint32) for x in (qid, threshold, length, ids, counts)]
        return int(self.L.or_hash_results(Q, _p(a[0], C.c_uint32), _p(a[1], C.c_uint32), _p(a[2], C.c_uint32),
                                          stride, _p(a[3], C.c_uint32), _p(a[4], C.c_uint32)))

    def lsh_params(self, family, m, dims, seed, w=4.0, sigma=1.0):
        d = max(dims, 1)
        a = np.zeros(m * d)
        b = np.zeros(m if family == 0 else m * d)
        hs, rs = np.zeros(m, np.uint64), np.zeros(m, np.uint64)
        self.L.or_lsh_params(family, m, dims, seed, w, sigma, _p(a, C.c_double), _p(b, C.c_double),
                             _p(hs, C.c_uint64), _p(rs, C.c_uint64))
        return a, b, hs, rs

    def lsh_encode(self, family, m, dims, seed, points=None, set_off=None, elems=None, w=4.0, sigma=1.0,
                   bucket_count=67, bucket_min=-33, rehash=False, domain=8192, nthreads=None):
        a, b, hs, rs = self.lsh_params(family, m, dims, seed, w, sigma)
        if family == 2:
            so = np.ascontiguousarray(set_off, np.uint64)
            el = np.ascontiguousarray(elems, np.uint64)
            n = so.shape[0] - 1
            pts = np.zeros(1, np.float32)
        else:
            pts = np.ascontiguousarray(points, np.float32)
            n = pts.shape[0]
            so, el = np.zeros(1, np.uint64), np.zeros(1, np.uint64)
        out = np.zeros((n, m), np.uint32)
        self.L.or_lsh_encode(family, m, dims, _p(a, C.c_double), _p(b, C.c_double), w, bucket_count, bucket_min,
                             int(rehash), _p(hs, C.c_uint64), _p(rs, C.c_uint64), domain, _p(pts, C.c_float),
                             _p(so, C.c_uint64), _p(el, C.c_uint64), n, nthreads or threads(), _p(out, C.c_uint32))
        return out

    def kernel_width(self, points, max_pairs=1_000_000):
        pts = np.ascontiguousarray(points, np.float32)
        return float(self.L.or_kernel_width(_p(pts, C.c_float), pts.shape[0], pts.shape[1], max_pairs))


class OracleIndex:
    def __init__(self, oracle: Oracle, csr):
        self.o = oracle
        self.csr = csr  # keep the arrays alive
        self.h = oracle.L.or_index_create(csr.n, csr.num_keys, _p(csr.keys, C.c_uint64), _p(csr.key_off, C.c_uint64),
                                          _p(csr.postings, C.c_uint32))

    def __del__(self):
        try:
            self.o.L.or_index_free(self.h)
        except Exception:
            pass

    def max_multiplicity(self, dim: int) -> int:
        return int(self.o.L.or_max_multiplicity(self.h, dim))

    def execute(self, batch, stride=None, nthreads=None):
        Q = len(batch)
        stride = int(stride or max(batch.max_k, 1))
        ids, counts = np.zeros((Q, stride), np.uint32), np.zeros((Q, stride), np.uint32)
        ln, thr = np.zeros(Q, np.uint32), np.zeros(Q, np.uint32)
        bound, post = np.zeros(Q, np.uint64), np.zeros(Q, np.uint64)
        bad = C.c_uint32()
        rc = self.o.L.or_execute(self.h, Q, _p(batch.qid, C.c_uint32), _p(batch.k, C.c_uint32),
                                 _p(batch.item_off, C.c_uint64), _p(batch.dim, C.c_uint16), _p(batch.lo, C.c_uint32),
                                 _p(batch.hi, C.c_uint32), stride, _p(ids, C.c_uint32), _p(counts, C.c_uint32),
                                 _p(ln, C.c_uint32), _p(thr, C.c_uint32), _p(bound, C.c_uint64), _p(post, C.c_uint64),
                                 nthreads or threads(), C.byref(bad))
        if rc:
            raise RuntimeError(f"oracle: status {rc} on query index {bad.value}")
        return OracleResult(batch.qid.copy(), ids, counts, ln, thr, bound, post)


class RefLib:
    """The reference itself (unmodified headers) behind oracle/ref_shim.cpp."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"reference shim not built: {path} (make -C oracle ref)")
        L = C.CDLL(str(path))
        E = (C.c_char_p, C.c_size_t)
        L.mcxref_hardware_threads.restype = C.c_uint
        L.mcxref_index_from_csr.argtypes = [C.c_uint32, C.c_uint64, u64p, u64p, u32p, C.c_uint32, C.POINTER(vp), *E]
        L.mcxref_index_from_objects.argtypes = [C.c_uint32, u64p, u16p, u32p, C.c_uint32, C.POINTER(vp), *E]
        L.mcxref_index_free.argtypes = [vp]
        L.mcxref_index_shape.argtypes = [vp, u64p, u64p, u64p]
        L.mcxref_index_export.argtypes = [vp, u64p, u32p, u16p, u64p, u64p, u32p]
        L.mcxref_max_multiplicity.restype = C.c_uint32
        L.mcxref_max_multiplicity.argtypes = [vp, C.c_uint16]
        L.mcxref_max_count_bound.argtypes = [vp, C.c_uint32, u16p, u32p, u32p, u64p, *E]
        L.mcxref_execute.argtypes = [vp, C.c_uint32, u32p, u32p, u64p, u16p, u32p, u32p, C.c_int, C.c_int, C.c_uint32,
                                     C.c_uint32, C.c_uint32, C.c_uint32, u32p, u32p, u32p, u32p, u64p, u64p, u64p, *E]
        L.mcxref_execute_partitioned.argtypes = [vp, C.c_uint32, C.c_uint32, u32p, u32p, u64p, u16p, u32p, u32p,
                                                 C.c_int, C.c_uint32, u32p, u32p, u32p, u32p, u64p, *E]
        L.mcxref_merge_topk.argtypes = [C.c_uint32, u64p, u32p, u32p, C.c_uint32, C.c_uint32, C.c_uint32, u32p, u32p,
                                        u32p, u32p, *E]
        L.mcxref_cpq_stream.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, u32p, C.c_uint32, u32p, u32p,
                                        u32p, u32p, u32p, *E]
        L.mcxref_mix64.restype, L.mcxref_mix64.argtypes = C.c_uint64, [C.c_uint64]
        L.mcxref_lsh_encode.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_double, C.c_uint32,
                                        C.c_int64, C.c_int, C.c_double, f32p, C.c_uint64, C.c_uint32, u32p, *E]
        L.mcxref_lsh_params.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_double, C.c_double, f64p,
                                        f64p, u64p, *E]
        L.mcxref_edit_distance_bounded.restype = C.c_uint32
        L.mcxref_edit_distance_bounded.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, C.c_uint32,
                                                   C.c_int]
        L.mcxref_verify_candidates.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, u32p, u32p, C.c_uint32,
                                               C.c_char_p, u64p, C.c_uint64, C.c_uint64, C.c_int, u32p, u32p,
                                               C.POINTER(C.c_int), u32p, C.POINTER(C.c_int64), *E]
        L.mcxref_kernel_width.restype = C.c_double
        L.mcxref_kernel_width.argtypes = [f32p, C.c_uint64, C.c_uint32, C.c_uint64]
        L.mcxref_index_serialize.argtypes = [vp, vp, u64p, *E]
        L.mcxref_deserialize.argtypes = [vp, C.c_uint64, *E]
        L.mcxref_hash_results.restype = C.c_uint64
        L.mcxref_hash_results.argtypes = [C.c_uint32, u32p, u32p, u32p, C.c_uint32, u32p, u32p]
        self.L = L

    def deserialize_status(self, image: bytes):
        """(status, message) deserialize_index (index_io.hpp:84-146) gives an image."""
        buf = (C.c_uint8 * max(1, len(image))).from_buffer_copy(image or b"\0")
        err = C.create_string_buffer(512)
        rc = self.L.mcxref_deserialize(C.cast(buf, vp), len(image), err, 512)
        return rc, err.value.decode()

    def hardware_threads(self) -> int:
        return int(self.L.mcxref_hardware_threads())

    @staticmethod
    def _check(rc, err):
        if rc:
            raise RuntimeError(f"reference error {rc}: {err.value.decode(errors='replace')}")

    def index(self, csr, split: int = 0) -> "RefIndex":
        h, err = vp(), C.create_string_buffer(1024)
        rc = self.L.mcxref_index_from_csr(csr.n, csr.num_keys, _p(csr.keys, C.c_uint64), _p(csr.key_off, C.c_uint64),
                                          _p(csr.postings, C.c_uint32), split, C.byref(h), err, len(err))
        self._check(rc, err)
        return RefIndex(self, h)

    def index_from_objects(self, n, obj_off, dims, tokens, split: int = 0) -> "RefIndex":
        obj_off = np.ascontiguousarray(obj_off, np.uint64)
        dims = np.ascontiguousarray(dims, np.uint16)
        tokens = np.ascontiguousarray(tokens, np.uint32)
        h, err = vp(), C.create_string_buffer(1024)
        rc = self.L.mcxref_index_from_objects(n, _p(obj_off, C.c_uint64), _p(dims, C.c_uint16),
                                              _p(tokens, C.c_uint32), split, C.byref(h), err, len(err))
        self._check(rc, err)
        return RefIndex(self, h)

    def cpq_stream(self, n, max_count, k, stream):
        s = np.ascontiguousarray(stream, np.uint32)
        cap = max(1, min(k, n) + k)
        ids, counts = np.zeros(cap, np.uint32), np.zeros(cap, np.uint32)
        ln, thr, at = C.c_uint32(), C.c_uint32(), C.c_uint32()
        err = C.create_string_buffer(512)
        rc = self.L.mcxref_cpq_stream(n, max_count, k, s.shape[0], _p(s, C.c_uint32), cap, _p(ids, C.c_uint32),
                                      _p(counts, C.c_uint32), C.byref(ln), C.byref(thr), C.byref(at), err, len(err))
        return rc, list(zip(ids[: ln.value].tolist(), counts[: ln.value].tolist())), thr.value, at.value

    def merge_topk(self, lists, k, query_id=0):
        off = np.zeros(len(lists) + 1, np.uint64)
        ids, counts = [], []
        for i, l in enumerate(lists):
            off[i + 1] = off[i] + len(l)
            ids += [e[0] for e in l]
            counts += [e[1] for e in l]
        ia, ca = np.array(ids + [0], np.uint32), np.array(counts + [0], np.uint32)
        cap = max(1, int(off[-1]))
        oi, oc = np.zeros(cap, np.uint32), np.zeros(cap, np.uint32)
        ln, thr = C.c_uint32(), C.c_uint32()
        err = C.create_string_buffer(512)
        rc = self.L.mcxref_merge_topk(len(lists), _p(off, C.c_uint64), _p(ia, C.c_uint32), _p(ca, C.c_uint32), k,
                                      query_id, cap, _p(oi, C.c_uint32), _p(oc, C.c_uint32), C.byref(ln),
                                      C.byref(thr), err, len(err))
        return rc, list(zip(oi[: ln.value].tolist(), oc[: ln.value].tolist())), thr.value

    def lsh_encode(self, family, m, dims, seed, points, w=4.0, sigma=1.0, bucket_count=67, bucket_min=-33,
                   rehash=False, domain=8192, nthreads=None):
        pts = np.ascontiguousarray(points, np.float32)
        n = pts.shape[0]
        out = np.zeros((n, m), np.uint32)
        err = C.create_string_buffer(512)
        rc = self.L.mcxref_lsh_encode(family, m, dims, seed, domain, w, bucket_count, bucket_min, int(rehash), sigma,
                                      _p(pts, C.c_float), n, nthreads or threads(), _p(out, C.c_uint32), err, len(err))
        self._check(rc, err)
        return out

    def lsh_params(self, family, m, dims, seed, w=4.0, sigma=1.0):
        a = np.zeros(m * dims)
        b = np.zeros(m if family == 0 else m * dims)
        rs = np.zeros(m, np.uint64)
        err = C.create_string_buffer(512)
        rc = self.L.mcxref_lsh_params(family, m, dims, seed, w, sigma, _p(a, C.c_double), _p(b, C.c_double),
                                      _p(rs, C.c_uint64), err, len(err))
        self._check(rc, err)
        return a, b, rs

    def kernel_width(self, points, max_pairs=1_000_000):
        pts = np.ascontiguousarray(points, np.float32)
        return float(self.L.mcxref_kernel_width(_p(pts, C.c_float), pts.shape[0], pts.shape[1], max_pairs))

    def edit_distance(self, a: bytes, b: bytes, cap=None) -> int:
        return int(self.L.mcxref_edit_distance_bounded(a, len(a), b, len(b), cap or 0, int(cap is not None)))

    def verify_candidates(self, query: bytes, ids, counts, n, corpus, requested_k=0, early_break=True):
        ids = np.ascontiguousarray(ids, np.uint32)
        counts = np.ascontiguousarray(counts, np.uint32)
        off = np.zeros(len(corpus) + 1, np.uint64)
        off[1:] = np.cumsum([len(c) for c in corpus])
        blob = b"".join(corpus)
        bi, bd, used = C.c_uint32(), C.c_uint32(), C.c_uint32()
        cert, theta = C.c_int(), C.c_int64()
        err = C.create_string_buffer(512)
        rc = self.L.mcxref_verify_candidates(query, len(query), ids.shape[0], _p(ids, C.c_uint32),
                                             _p(counts, C.c_uint32), n, blob, _p(off, C.c_uint64), len(corpus),
                                             requested_k, int(early_break), C.byref(bi), C.byref(bd), C.byref(cert),
                                             C.byref(used), C.byref(theta), err, len(err))
        self._check(rc, err)
        return bi.value, bd.value, bool(cert.value), used.value, theta.value


# ---- sequence search restated in plain Python (sa.hpp), small cases only

def edit_distance(a: bytes, b: bytes) -> int:
    """sa.hpp:109-123: unit-cost Levenshtein distance, two-row DP."""
    if len(a) < len(b):
        a, b = b, a
    row = list(range(len(b) + 1))
    for i in range(1, len(a) + 1):
        diag, row[0] = row[0], i
        for j in range(1, len(b) + 1):
            up = row[j]
            row[j] = min(up + 1, row[j - 1] + 1, diag + (a[i - 1] != b[j - 1]))
            diag = up
    return row[len(b)]


def edit_distance_bounded(a: bytes, b: bytes, cap: int) -> int:
    """sa.hpp:127-162: the exact distance when <= cap, else cap + 1."""
    if abs(len(a) - len(b)) > cap:
        return cap + 1
    return min(edit_distance(a, b), cap + 1)


def verify_candidates(query: bytes, hits, n: int, corpus, requested_k: int = 0, early_break: bool = True,
                      dist=None):
    """sa.hpp:298-336.  hits: [(id, count)] by descending count.  `dist(id, cap)`
    supplies bounded distances (default: the DP above).  Returns (best_id,
    best_distance, certified, candidates_used, threshold_at_stop)."""
    if not hits:
        raise ValueError("verify_candidates: empty candidate list")
    dist = dist or (lambda i, cap: edit_distance(query, corpus[i]) if cap is None
                    else edit_distance_bounded(query, corpus[i], cap))
    requested_k = requested_k or len(hits)
    qlen = len(query)
    best_id = hits[0][0]
    best = dist(best_id, None)  # cap None: the exact distance (edit_distance)
    used = 1
    theta = qlen - n + 1 - n * (best - 1)
    for cid, cnt in hits[1:]:
        if early_break and theta > cnt:
            break
        used += 1
        if abs(len(corpus[cid]) - qlen) > best or best == 0:
            continue
        d = dist(cid, best - 1)
        if d < best:
            best_id, best = cid, d
            theta = qlen - n + 1 - n * (d - 1)
    c_k = hits[-1][1] if len(hits) >= requested_k else 0
    certified = c_k < qlen - n + 1 - best * n
    return best_id, best, certified, used, theta


class RefIndex:
    def __init__(self, lib: RefLib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            self.lib.L.mcxref_index_free(self.h)
        except Exception:
            pass

    def serialize(self) -> bytes:
        """serialize_index (index_io.hpp:63-82) of the reference index."""
        L = self.lib.L
        size, err = C.c_uint64(0), C.create_string_buffer(512)
        RefLib._check(L.mcxref_index_serialize(self.h, None, C.byref(size), err, 512), err)
        out = (C.c_uint8 * max(1, size.value))()
        RefLib._check(L.mcxref_index_serialize(self.h, C.cast(out, vp), C.byref(size), err, 512), err)
        return bytes(out)[: size.value]

    def shape(self):
        K, P, S = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.lib.L.mcxref_index_shape(self.h, C.byref(K), C.byref(P), C.byref(S))
        return K.value, P.value, S.value

    def export(self):
        K, P, S = self.shape()
        keys, first, cnt = np.zeros(K, np.uint64), np.zeros(K, np.uint32), np.zeros(K, np.uint16)
        sb, se, post = np.zeros(S, np.uint64), np.zeros(S, np.uint64), np.zeros(P, np.uint32)
        self.lib.L.mcxref_index_export(self.h, _p(keys, C.c_uint64), _p(first, C.c_uint32), _p(cnt, C.c_uint16),
                                       _p(sb, C.c_uint64), _p(se, C.c_uint64), _p(post, C.c_uint32))
        return keys, first, cnt, sb, se, post

    def max_multiplicity(self, dim):
        return int(self.lib.L.mcxref_max_multiplicity(self.h, dim))

    def max_count_bound(self, dim, lo, hi):
        d, l, h = (np.ascontiguousarray(x, t) for x, t in ((dim, np.uint16), (lo, np.uint32), (hi, np.uint32)))
        out, err = C.c_uint64(), C.create_string_buffer(512)
        rc = self.lib.L.mcxref_max_count_bound(self.h, d.shape[0], _p(d, C.c_uint16), _p(l, C.c_uint32),
                                               _p(h, C.c_uint32), C.byref(out), err, len(err))
        RefLib._check(rc, err)
        return out.value

    def execute(self, batch, selector=0, sequential=False, workers=0, span_chunk=4096, spans_per_task=2,
                stride=None):
        Q = len(batch)
        stride = int(stride or max(batch.max_k, 1))
        ids, counts = np.zeros((Q, stride), np.uint32), np.zeros((Q, stride), np.uint32)
        ln, thr = np.zeros(Q, np.uint32), np.zeros(Q, np.uint32)
        h = C.c_uint64()
        t5, m3 = np.zeros(5, np.uint64), np.zeros(3, np.uint64)
        err = C.create_string_buffer(1024)
        rc = self.lib.L.mcxref_execute(self.h, Q, _p(batch.qid, C.c_uint32), _p(batch.k, C.c_uint32),
                                       _p(batch.item_off, C.c_uint64), _p(batch.dim, C.c_uint16),
                                       _p(batch.lo, C.c_uint32), _p(batch.hi, C.c_uint32), selector,
                                       1 if sequential else 0, workers, span_chunk, spans_per_task, stride,
                                       _p(ids, C.c_uint32), _p(counts, C.c_uint32), _p(ln, C.c_uint32),
                                       _p(thr, C.c_uint32), C.byref(h), _p(t5, C.c_uint64), _p(m3, C.c_uint64), err,
                                       len(err))
        if rc:
            return rc, err.value.decode(errors="replace")
        r = OracleResult(batch.qid.copy(), ids, counts, ln, thr)
        r.hash = h.value
        r.timings = dict(zip(("lookup_ns", "match_ns", "select_ns", "merge_ns", "total_ns"), t5.tolist()))
        r.memory = dict(zip(("counter_bytes", "gate_bytes", "table_bytes"), m3.tolist()))
        return 0, r

    def execute_partitioned(self, batch, capacity, sequential=True, stride=None):
        Q = len(batch)
        stride = int(stride or max(batch.max_k, 1))
        ids, counts = np.zeros((Q, stride), np.uint32), np.zeros((Q, stride), np.uint32)
        ln, thr = np.zeros(Q, np.uint32), np.zeros(Q, np.uint32)
        h = C.c_uint64()
        err = C.create_string_buffer(1024)
        rc = self.lib.L.mcxref_execute_partitioned(self.h, capacity, Q, _p(batch.qid, C.c_uint32),
                                                   _p(batch.k, C.c_uint32), _p(batch.item_off, C.c_uint64),
                                                   _p(batch.dim, C.c_uint16), _p(batch.lo, C.c_uint32),
                                                   _p(batch.hi, C.c_uint32), 1 if sequential else 0, stride,
                                                   _p(ids, C.c_uint32), _p(counts, C.c_uint32), _p(ln, C.c_uint32),
                                                   _p(thr, C.c_uint32), C.byref(h), err, len(err))
        if rc:
            return rc, err.value.decode(errors="replace")
        r = OracleResult(batch.qid.copy(), ids, counts, ln, thr)
        r.hash = h.value
        return 0, r


def ref_available() -> bool:
    return REF_SO.exists()
