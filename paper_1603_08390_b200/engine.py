"""Array-level host API over the C ABI (the layer bench.py and the tests use).

`DeviceIndex` owns one `genie_index` (a CSR inverted index resident in HBM on
one GPU) and runs batches of match-count queries through the hand-written
sm_100a pipeline.  Inputs and outputs are numpy arrays (host API) or torch
CUDA tensors (device API).  The object-level mirror of the reference API
(`mcx.py`) is built on top of this module.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N


# ---------------------------------------------------------------- errors
# mcx/error.hpp:24-41


class McxError(Exception):
    pass


class ContractError(McxError, ValueError):
    """A caller broke a documented precondition (mcx::ContractError)."""


class DataError(McxError, RuntimeError):
    """Malformed input data (mcx::DataError)."""


class InvariantError(McxError, RuntimeError):
    """An internal invariant failed (mcx::InvariantError)."""


class CudaError(McxError, RuntimeError):
    """CUDA / device failure."""


_ERRORS = {
    N.GENIE_ERR_CONTRACT: ContractError,
    N.GENIE_ERR_DATA: DataError,
    N.GENIE_ERR_INVARIANT: InvariantError,
    N.GENIE_ERR_CUDA: CudaError,
    N.GENIE_ERR_NCCL: CudaError,
}


def check(rc: int, err: C.Array) -> None:
    if rc != N.GENIE_OK:
        raise _ERRORS.get(rc, McxError)(err.value.decode(errors="replace"))


def _errbuf() -> C.Array:
    return C.create_string_buffer(1024)


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


# ----------------------------------------------------------------- inputs


def _torch_stream(stream: Optional[int]) -> C.c_void_p:
    """The CUDA stream a device-array call is ordered on: the given handle, or
    torch's current stream -- so work queued on torch tensors (uploads, fills)
    is complete before the kernels read them.  torch's legacy default stream
    has handle 0, which the C ABI reads as "the handle's own stream"; it is
    passed as cudaStreamLegacy (0x1) instead."""
    if stream is None:
        import torch

        stream = torch.cuda.current_stream().cuda_stream
    return C.c_void_p(stream if stream else 1)


@dataclass
class CSR:
    """Host CSR inverted index: keys (packed dim<<32|token, ascending),
    key_off[K+1], postings (ascending ids per key).  The layout of
    InvertedIndex's position map + list array (index.hpp:41-182) without
    sub-list splitting."""

    n: int
    keys: np.ndarray
    key_off: np.ndarray
    postings: np.ndarray

    def __post_init__(self):
        self.keys = np.ascontiguousarray(self.keys, dtype=np.uint64)
        self.key_off = np.ascontiguousarray(self.key_off, dtype=np.uint64)
        self.postings = np.ascontiguousarray(self.postings, dtype=np.uint32)

    @property
    def num_keys(self) -> int:
        return int(self.keys.shape[0])

    @property
    def num_postings(self) -> int:
        return int(self.postings.shape[0])


@dataclass
class QueryBatch:
    """Queries as flat arrays: query q owns items [item_off[q], item_off[q+1])."""

    qid: np.ndarray
    k: np.ndarray
    item_off: np.ndarray
    dim: np.ndarray
    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self):
        self.qid = np.ascontiguousarray(self.qid, dtype=np.uint32)
        self.k = np.ascontiguousarray(self.k, dtype=np.uint32)
        self.item_off = np.ascontiguousarray(self.item_off, dtype=np.uint64)
        self.dim = np.ascontiguousarray(self.dim, dtype=np.uint16)
        self.lo = np.ascontiguousarray(self.lo, dtype=np.uint32)
        self.hi = np.ascontiguousarray(self.hi, dtype=np.uint32)

    def __len__(self) -> int:
        return int(self.qid.shape[0])

    @property
    def max_k(self) -> int:
        return int(self.k.max()) if len(self) else 0

    @property
    def num_items(self) -> int:
        return int(self.item_off[-1] - self.item_off[0]) if len(self) else 0

    def slice(self, a: int, b: int) -> "QueryBatch":
        i0, i1 = int(self.item_off[a]), int(self.item_off[b])
        return QueryBatch(self.qid[a:b], self.k[a:b], self.item_off[a : b + 1] - i0, self.dim[i0:i1],
                          self.lo[i0:i1], self.hi[i0:i1])

    def nbytes(self) -> int:
        return sum(int(x.nbytes) for x in (self.qid, self.k, self.item_off, self.dim, self.lo, self.hi))


@dataclass
class Results:
    """TopKResult rows: row q holds length[q] entries (count desc, id asc)."""

    qid: np.ndarray
    ids: np.ndarray  # [Q, stride] uint32
    counts: np.ndarray  # [Q, stride] uint32
    length: np.ndarray
    threshold: np.ndarray
    bound: Optional[np.ndarray] = None
    timings: Optional[dict] = None
    stats: Optional[dict] = None

    def row(self, q: int):
        n = int(self.length[q])
        return list(zip(self.ids[q, :n].tolist(), self.counts[q, :n].tolist()))

    def hash(self) -> int:
        return hash_results(self.qid, self.threshold, self.length, self.ids, self.counts)


def config(selector: int = 0, span_chunk: Optional[int] = None, max_spans_per_task: int = 2,
           tile_bytes: int = 0, ctas_per_sm: int = 0, stage_events: bool = False, graph: bool = False) -> N.Config:
    c = N.engine().genie_config_default()
    c.flags = (N.GENIE_FLAG_STAGE_EVENTS if stage_events else 0) | (N.GENIE_FLAG_GRAPH if graph else 0)
    c.selector = selector
    if span_chunk is not None:
        c.span_chunk = span_chunk
    c.max_spans_per_task = max_spans_per_task
    c.tile_bytes = tile_bytes
    c.ctas_per_sm = ctas_per_sm
    return c


def hash_results(qid, threshold, length, ids, counts) -> int:
    """engine.hpp:141-153 over result arrays."""
    Q = int(len(qid))
    stride = int(ids.shape[1]) if ids.ndim == 2 and Q else 0
    ent = np.zeros((Q, max(stride, 1), 2), dtype=np.uint32)
    if stride:
        ent[:, :stride, 0] = ids
        ent[:, :stride, 1] = counts
    qid = np.ascontiguousarray(qid, dtype=np.uint32)
    thr = np.ascontiguousarray(threshold, dtype=np.uint32)
    ln = np.ascontiguousarray(length, dtype=np.uint32)
    return int(N.engine().genie_hash_results(Q, _ptr(qid, C.c_uint32), _ptr(thr, C.c_uint32),
                                             _ptr(ln, C.c_uint32), max(stride, 1),
                                             ent.ctypes.data_as(C.POINTER(N.Entry))))


# ------------------------------------------------------------------ index


class DeviceIndex:
    """One GPU's inverted index (a `genie_index` handle)."""

    def __init__(self, handle: int, lib=None):
        self._h = C.c_void_p(handle)
        self._lib = lib or N.engine()
        n, K, P, off, dev = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_int()
        self._lib.genie_index_info(self._h, C.byref(n), C.byref(K), C.byref(P), C.byref(off), C.byref(dev))
        self.num_objects, self.num_keys, self.num_postings = n.value, K.value, P.value
        self.id_offset, self.device = off.value, dev.value

    # construction ------------------------------------------------------
    @classmethod
    def from_csr(cls, csr: CSR, device: int = 0, id_offset: int = 0,
                 dim_max_mult: Optional[np.ndarray] = None) -> "DeviceIndex":
        lib = N.engine()
        h, err = C.c_void_p(), _errbuf()
        dm = None
        if dim_max_mult is not None:
            dm = np.ascontiguousarray(dim_max_mult, dtype=np.uint32)
            assert dm.shape == (65536,)
        key_off = csr.key_off if csr.key_off.size else np.zeros(1, np.uint64)
        rc = lib.genie_index_create(csr.n, csr.num_keys, _ptr(csr.keys, C.c_uint64), _ptr(key_off, C.c_uint64),
                                    _ptr(csr.postings, C.c_uint32), None if dm is None else _ptr(dm, C.c_uint32),
                                    id_offset, device, C.byref(h), err, len(err))
        check(rc, err)
        return cls(h.value, lib)

    @classmethod
    def build(cls, n: int, obj_off: np.ndarray, dims: np.ndarray, tokens: np.ndarray,
              device: int = 0) -> "DeviceIndex":
        """build_index (index.hpp:190-250) on the device: object o owns
        keywords [obj_off[o], obj_off[o+1]) of dims/tokens."""
        off = np.ascontiguousarray(obj_off, np.uint64)
        d = np.ascontiguousarray(dims, np.uint16)
        t = np.ascontiguousarray(tokens, np.uint32)
        assert off.shape == (n + 1,) and d.shape == t.shape
        lib = N.engine()
        h, err = C.c_void_p(), _errbuf()
        d1 = d if d.size else np.zeros(1, np.uint16)
        t1 = t if t.size else np.zeros(1, np.uint32)
        check(lib.genie_index_build(n, _ptr(off, C.c_uint64), _ptr(d1, C.c_uint16), _ptr(t1, C.c_uint32), device,
                                    C.byref(h), err, len(err)), err)
        return cls(h.value, lib)

    @classmethod
    def from_mcix(cls, image, device: int = 0) -> "DeviceIndex":
        """load_index (index_io.hpp:148-154): an MCIX image (bytes or a path)
        validated like deserialize_index and uploaded as the device CSR."""
        data = _mcix_bytes(image)
        lib = N.engine()
        h, err = C.c_void_p(), _errbuf()
        buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data or b"\0")
        check(lib.genie_index_load_mcix(C.cast(buf, C.c_void_p), len(data), device, C.byref(h), err, len(err)), err)
        return cls(h.value, lib)

    @classmethod
    def shard(cls, csr: CSR, id_begin: int, id_end: int, device: int = 0) -> "DeviceIndex":
        """Object-id range [id_begin, id_end) of a full CSR (one partition of
        partition_dataset, index.hpp:263-291), ids rebased, offset kept."""
        lib = N.engine()
        h, err = C.c_void_p(), _errbuf()
        rc = lib.genie_index_create_shard(csr.n, csr.num_keys, _ptr(csr.keys, C.c_uint64),
                                          _ptr(csr.key_off, C.c_uint64), _ptr(csr.postings, C.c_uint32),
                                          id_begin, id_end, device, C.byref(h), err, len(err))
        check(rc, err)
        return cls(h.value, lib)

    @classmethod
    def from_tokens_device(cls, d_tokens_ptr: int, n: int, m: int, domain: int, device: int = 0,
                           id_offset: int = 0) -> "DeviceIndex":
        lib = N.engine()
        h, err = C.c_void_p(), _errbuf()
        rc = lib.genie_index_from_tokens_device(C.c_void_p(d_tokens_ptr), n, m, domain, id_offset, device,
                                                C.byref(h), err, len(err))
        check(rc, err)
        return cls(h.value, lib)

    def close(self):
        if self._h and self._h.value:
            self._lib.genie_index_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    # facts -----------------------------------------------------------------
    def dim_stats(self) -> np.ndarray:
        out = np.zeros(65536, np.uint32)
        err = _errbuf()
        check(self._lib.genie_index_dim_stats(self._h, _ptr(out, C.c_uint32), err, len(err)), err)
        return out

    def export(self) -> CSR:
        keys = np.zeros(self.num_keys, np.uint64)
        off = np.zeros(self.num_keys + 1, np.uint64)
        post = np.zeros(self.num_postings, np.uint32)
        err = _errbuf()
        check(self._lib.genie_index_export(self._h, _ptr(keys, C.c_uint64), _ptr(off, C.c_uint64),
                                           _ptr(post, C.c_uint32), err, len(err)), err)
        return CSR(self.num_objects, keys, off, post)

    # queries -----------------------------------------------------------------
    def query(self, batch: QueryBatch, cfg: Optional[N.Config] = None, stride: Optional[int] = None,
              timings: bool = False, want_bound: bool = False, out=None, copy: bool = True) -> Results:
        """execute_batch (engine.hpp:184-304) with host buffers.  `out` may hold
        preallocated (pinned) result buffers (entries [Q, stride, 2] u32, length
        [Q] u32, threshold [Q] u32)."""
        Q = len(batch)
        stride = int(stride if stride is not None else max(min(batch.max_k, self.num_objects), 1))
        if out is not None:
            ent, ln, thr = out
            assert ent.shape == (Q, stride, 2) and ent.dtype == np.uint32 and ent.flags.c_contiguous
        else:
            ent = np.zeros((Q, stride, 2), dtype=np.uint32)
            ln = np.zeros(Q, np.uint32)
            thr = np.zeros(Q, np.uint32)
        bound = np.zeros(Q, np.uint64) if want_bound else None
        st = N.StageNs()
        stats = N.BatchStats()
        err = _errbuf()
        cfg = cfg if cfg is not None else config()
        rc = self._lib.genie_query_batch(
            self._h, C.byref(cfg), Q, batch.qid.ctypes.data, batch.k.ctypes.data, batch.item_off.ctypes.data,
            batch.dim.ctypes.data, batch.lo.ctypes.data, batch.hi.ctypes.data, stride, ent.ctypes.data,
            ln.ctypes.data, thr.ctypes.data, None if bound is None else bound.ctypes.data,
            C.byref(st) if timings else None, C.byref(stats), err, len(err))
        check(rc, err)
        tdict = {f: getattr(st, f) for f, _ in N.StageNs._fields_} if timings else None
        sdict = {f: getattr(stats, f) for f, _ in N.BatchStats._fields_}
        if not copy:
            return Results(batch.qid, ent[:, :, 0], ent[:, :, 1], ln, thr, bound, tdict, sdict)
        return Results(batch.qid.copy(), ent[:, :, 0].copy(), ent[:, :, 1].copy(), ln, thr, bound, tdict, sdict)

    def stage_ns(self) -> dict:
        """Device stage times of the last batch launched with stage events."""
        st, err = N.StageNs(), _errbuf()
        check(self._lib.genie_last_stage_ns(self._h, C.byref(st), err, len(err)), err)
        return {f: getattr(st, f) for f, _ in N.StageNs._fields_}

    def query_device(self, d: dict, cfg: Optional[N.Config] = None, stream: Optional[int] = None) -> int:
        """Enqueue a batch whose arrays are torch CUDA tensors in `d` (keys qid,
        k, item_off, dim, lo, hi, out, out_len, out_thr; ints max_k,
        total_items, stride).  Returns the number of kernels launched.  Call
        `status()` after synchronising."""
        err = _errbuf()
        cfg = cfg if cfg is not None else config()
        ptr = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        rc = self._lib.genie_query_batch_device(
            self._h, C.byref(cfg), int(d["qid"].numel()), ptr(d["qid"]), ptr(d["k"]), ptr(d["item_off"]),
            ptr(d["dim"]), ptr(d["lo"]), ptr(d["hi"]), int(d["max_k"]), int(d["total_items"]), int(d["stride"]),
            ptr(d["out"]), ptr(d["out_len"]), ptr(d["out_thr"]), _torch_stream(stream), err, len(err))
        check(rc, err)
        return int(self._lib.genie_last_launch_count(self._h))

    def graph_captures(self) -> int:
        return int(self._lib.genie_graph_captures(self._h))

    def status(self) -> dict:
        """Synchronise and surface the last device batch's status; raises on
        errors, returns "retry" when the workspace had to grow."""
        stats = N.BatchStats()
        err = _errbuf()
        rc = self._lib.genie_query_status(self._h, C.byref(stats), err, len(err))
        if rc == N.GENIE_RETRY:
            return {"retry": True}
        check(rc, err)
        return {f: getattr(stats, f) for f, _ in N.BatchStats._fields_}

    def merge_device(self, Q: int, L: int, d_in, d_in_len, in_stride: int, d_k, stride: int, d_out, d_out_len,
                     d_out_thr, stream: Optional[int] = None, list_major: bool = False) -> None:
        """merge_topk over per-shard lists resident on this device (the
        multi-GPU combine step after an all-gather): lists query-major
        [Q, L, in_stride] or, with list_major, [L, Q, in_stride] -- the order
        an all-gather of per-shard rows produces."""
        err = _errbuf()
        ptr = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        rc = self._lib.genie_merge_topk_device_layout(self._h, Q, L, ptr(d_in), ptr(d_in_len), in_stride,
                                                      int(list_major), ptr(d_k), stride, ptr(d_out), ptr(d_out_len),
                                                      ptr(d_out_thr), _torch_stream(stream), err, len(err))
        check(rc, err)


class DeviceGroup:
    """Object-id-range shards of one index on several devices, driven by this
    one host thread (genie_group_*): every shard's batch runs at
    once, rows are exchanged (NCCL all-gather when the shards sit on distinct
    devices, peer copies otherwise) and merged on the first device."""

    def __init__(self, handle: int, lib, keep=()):
        self._h = C.c_void_p(handle)
        self._lib = lib
        self._keep = list(keep)  # borrowed DeviceIndex objects stay alive
        n, ex, no = C.c_uint32(), C.c_int(), C.c_uint32()
        lib.genie_group_info(self._h, C.byref(n), C.byref(ex), C.byref(no))
        self.num_shards, self.exchange, self.num_objects = n.value, ex.value, no.value

    @classmethod
    def from_csr(cls, csr: CSR, devices, exchange: int = N.GENIE_EXCHANGE_AUTO) -> "DeviceGroup":
        lib = N.engine()
        devs = (C.c_int * len(devices))(*devices)
        h, err = C.c_void_p(), _errbuf()
        key_off = csr.key_off if csr.key_off.size else np.zeros(1, np.uint64)
        check(lib.genie_group_create(csr.n, csr.num_keys, _ptr(csr.keys, C.c_uint64), _ptr(key_off, C.c_uint64),
                                     _ptr(csr.postings, C.c_uint32), len(devices), devs, exchange, C.byref(h), err,
                                     len(err)), err)
        return cls(h.value, lib)

    @classmethod
    def from_indexes(cls, indexes, id_offsets, exchange: int = N.GENIE_EXCHANGE_AUTO) -> "DeviceGroup":
        lib = N.engine()
        hs = (C.c_void_p * len(indexes))(*[ix.handle.value for ix in indexes])
        offs = np.ascontiguousarray(id_offsets, np.uint32)
        h, err = C.c_void_p(), _errbuf()
        check(lib.genie_group_from_indexes(hs, _ptr(offs, C.c_uint32), len(indexes), exchange, C.byref(h), err,
                                           len(err)), err)
        return cls(h.value, lib, keep=indexes)

    def close(self):
        if self._h and self._h.value:
            self._lib.genie_group_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def query(self, batch: QueryBatch, cfg: Optional[N.Config] = None, stride: Optional[int] = None,
              timings: bool = False) -> Results:
        Q = len(batch)
        stride = int(stride if stride is not None else max(min(batch.max_k, self.num_objects), 1))
        ent = np.zeros((Q, stride, 2), dtype=np.uint32)
        ln = np.zeros(Q, np.uint32)
        thr = np.zeros(Q, np.uint32)
        st, stats, err = N.StageNs(), N.BatchStats(), _errbuf()
        cfg = cfg if cfg is not None else config()
        rc = self._lib.genie_group_query_batch(
            self._h, C.byref(cfg), Q, _ptr(batch.qid, C.c_uint32), _ptr(batch.k, C.c_uint32),
            _ptr(batch.item_off, C.c_uint64), _ptr(batch.dim, C.c_uint16), _ptr(batch.lo, C.c_uint32),
            _ptr(batch.hi, C.c_uint32), stride, ent.ctypes.data_as(C.POINTER(N.Entry)), _ptr(ln, C.c_uint32),
            _ptr(thr, C.c_uint32), C.byref(st) if timings else None, C.byref(stats), err, len(err))
        check(rc, err)
        tdict = {f: getattr(st, f) for f, _ in N.StageNs._fields_} if timings else None
        sdict = {f: getattr(stats, f) for f, _ in N.BatchStats._fields_}
        return Results(batch.qid.copy(), ent[:, :, 0].copy(), ent[:, :, 1].copy(), ln, thr, None, tdict, sdict)


def merge_lists(lists_ids: np.ndarray, lists_counts: np.ndarray, lists_len: np.ndarray, k: np.ndarray,
                stride: Optional[int] = None, device: int = 0):
    """Batched merge_topk on the GPU: inputs [Q, L, S] ids/counts, [Q, L] lengths."""
    Q, L, S = lists_ids.shape
    k = np.ascontiguousarray(k, np.uint32)
    stride = int(stride if stride is not None else max(1, min(int(k.max()) if Q else 1, L * S)))
    inp = np.zeros((Q, L, S, 2), np.uint32)
    inp[..., 0] = lists_ids
    inp[..., 1] = lists_counts
    ln = np.ascontiguousarray(lists_len, np.uint32)
    out = np.zeros((Q, stride, 2), np.uint32)
    olen = np.zeros(Q, np.uint32)
    othr = np.zeros(Q, np.uint32)
    err = _errbuf()
    rc = N.engine().genie_merge_topk(device, Q, L, inp.ctypes.data_as(C.POINTER(N.Entry)), _ptr(ln, C.c_uint32), S,
                                     _ptr(k, C.c_uint32), stride, out.ctypes.data_as(C.POINTER(N.Entry)),
                                     _ptr(olen, C.c_uint32), _ptr(othr, C.c_uint32), err, len(err))
    check(rc, err)
    return out[..., 0].copy(), out[..., 1].copy(), olen, othr


# --------------------------------------------------------------------- LSH

PSTABLE, RBH, MINHASH = 0, 1, 2


class SeqSet:
    """A device-resident corpus of byte strings and the GPU edit-distance
    kernel over it (genie_seqset_*, sa.hpp:127-162): distances of a query to
    chosen sequences (or all of them), exact up to `cap`, cap + 1 beyond."""

    UNCAPPED = 0xFFFFFFFF

    def __init__(self, corpus, device: int = 0):
        seqs = [s if isinstance(s, bytes) else str(s).encode() for s in corpus]
        off = np.zeros(len(seqs) + 1, np.uint64)
        off[1:] = np.cumsum([len(s) for s in seqs])
        blob = np.frombuffer(b"".join(seqs) + b"\0", np.uint8)
        self._lib = N.engine()
        h, err = C.c_void_p(), _errbuf()
        check(self._lib.genie_seqset_create(C.c_void_p(blob.ctypes.data), _ptr(off, C.c_uint64), len(seqs), device,
                                            C.byref(h), err, len(err)), err)
        self._h = h
        self.lengths = np.diff(off).astype(np.int64)
        self.num_sequences = len(seqs)

    def close(self):
        if self._h and self._h.value:
            self._lib.genie_seqset_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def distances(self, query, ids=None, cap: int = UNCAPPED) -> np.ndarray:
        q = query if isinstance(query, bytes) else str(query).encode()
        qa = np.frombuffer(q + b"\0", np.uint8)
        idv = None if ids is None else np.ascontiguousarray(ids, np.uint32)
        count = self.num_sequences if idv is None else idv.shape[0]
        out = np.zeros(max(count, 1), np.uint32)
        err = _errbuf()
        check(self._lib.genie_seqset_distances(self._h, C.c_void_p(qa.ctypes.data), len(q),
                                               None if idv is None else _ptr(idv, C.c_uint32), count, cap,
                                               _ptr(out, C.c_uint32), err, len(err)), err)
        return out[:count]


def lsh_config(family: int = RBH, m: int = 237, dims: int = 0, seed: int = 1, rehash_domain: int = 8192,
               w: float = 4.0, bucket_count: int = 67, bucket_min: int = -33, rehash_pstable: bool = False,
               sigma: float = 1.0, fp32: bool = False) -> N.LshConfig:
    """LshEncoderConfig (lsh.hpp:132-145) defaults; fp32=True selects the
    opt-in fast transforms (not bit-exact, see genie.h)."""
    c = N.LshConfig()
    c.family, c.m, c.dims, c.seed = family, m, dims, seed
    c.rehash_domain, c.w, c.bucket_count, c.bucket_min = rehash_domain, w, bucket_count, bucket_min
    c.rehash_pstable, c.sigma = int(rehash_pstable), sigma
    c.precision = 1 if fp32 else 0
    return c


def lsh_sample(cfg: N.LshConfig):
    """Host-side parameters exactly as LshEncoder::create samples them."""
    m, d = cfg.m, max(cfg.dims, 1)
    if cfg.family == PSTABLE:
        a, b = np.zeros(m * d), np.zeros(m)
    elif cfg.family == RBH:
        a, b = np.zeros(m * d), np.zeros(m * d)
    else:
        a, b = np.zeros(1), np.zeros(1)
    hs, rs = np.zeros(m, np.uint64), np.zeros(m, np.uint64)
    err = _errbuf()
    check(N.engine().genie_lsh_sample(C.byref(cfg), _ptr(a, C.c_double), _ptr(b, C.c_double),
                                      _ptr(hs, C.c_uint64), _ptr(rs, C.c_uint64), err, len(err)), err)
    return a, b, hs, rs


class Encoder:
    """LshEncoder (lsh.hpp:149-219) with its transforms on the GPU."""

    def __init__(self, cfg: N.LshConfig, device: int = 0):
        self.cfg = cfg
        self.device = device
        self._lib = N.engine()
        h, err = C.c_void_p(), _errbuf()
        check(self._lib.genie_encoder_create(C.byref(cfg), device, C.byref(h), err, len(err)), err)
        self._h = h

    def close(self):
        if self._h and self._h.value:
            self._lib.genie_encoder_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def encode(self, points: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        pts = np.ascontiguousarray(points, dtype=np.float32)
        n = pts.shape[0]
        if out is None:
            out = np.zeros((n, self.cfg.m), np.uint32)
        assert out.shape == (n, self.cfg.m) and out.dtype == np.uint32 and out.flags.c_contiguous
        err = _errbuf()
        check(self._lib.genie_lsh_encode(self._h, _ptr(pts, C.c_float), n, _ptr(out, C.c_uint32), err, len(err)),
              err)
        return out

    def encode_device(self, d_points, d_tokens, stream: Optional[int] = None) -> None:
        err = _errbuf()
        check(self._lib.genie_lsh_encode_device(self._h, C.c_void_p(d_points.data_ptr()), int(d_points.shape[0]),
                                                C.c_void_p(d_tokens.data_ptr()), _torch_stream(stream), err,
                                                len(err)), err)

    def encode_sets(self, set_off: np.ndarray, elems: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        off = np.ascontiguousarray(set_off, np.uint64)
        el = np.ascontiguousarray(elems, np.uint64)
        n = off.shape[0] - 1
        if out is None:
            out = np.zeros((n, self.cfg.m), np.uint32)
        assert out.shape == (n, self.cfg.m) and out.dtype == np.uint32 and out.flags.c_contiguous
        err = _errbuf()
        check(self._lib.genie_minhash_encode(self._h, _ptr(off, C.c_uint64), _ptr(el, C.c_uint64), n,
                                             _ptr(out, C.c_uint32), err, len(err)), err)
        return out

    def encode_sets_device(self, d_off, d_elems, d_tokens, stream: Optional[int] = None) -> None:
        err = _errbuf()
        check(self._lib.genie_minhash_encode_device(self._h, C.c_void_p(d_off.data_ptr()),
                                                    C.c_void_p(d_elems.data_ptr()), int(d_off.shape[0]) - 1,
                                                    C.c_void_p(d_tokens.data_ptr()), _torch_stream(stream), err,
                                                    len(err)), err)

    def query(self, index: "DeviceIndex", k: int, points: Optional[np.ndarray] = None,
              set_off: Optional[np.ndarray] = None, elems: Optional[np.ndarray] = None, first_id: int = 0,
              cfg: Optional[N.Config] = None, stride: Optional[int] = None, out=None, copy: bool = True) -> Results:
        """encode_query_point + execute_batch in one GPU call (genie_lsh_query_batch):
        host points (or sets) in, results out; the tokens stay on the device."""
        if points is not None:
            pts = np.ascontiguousarray(points, np.float32)
            n, pp, so, el = pts.shape[0], pts.ctypes.data, None, None
        else:
            so = np.ascontiguousarray(set_off, np.uint64)
            el = np.ascontiguousarray(elems, np.uint64)
            n, pp = so.shape[0] - 1, None
        Q = int(n)
        stride = int(stride if stride is not None else max(min(k, index.num_objects), 1))
        if out is not None:
            ent, ln, thr = out
        else:
            ent, ln, thr = np.zeros((Q, stride, 2), np.uint32), np.zeros(Q, np.uint32), np.zeros(Q, np.uint32)
        stats, err = N.BatchStats(), _errbuf()
        cfg = cfg if cfg is not None else config()
        check(self._lib.genie_lsh_query_batch(
            self._h, index.handle, C.byref(cfg), pp, None if so is None else so.ctypes.data,
            None if el is None else el.ctypes.data, Q, k, first_id, stride, ent.ctypes.data, ln.ctypes.data,
            thr.ctypes.data, C.byref(stats), err, len(err)), err)
        qid = np.arange(first_id, first_id + Q, dtype=np.uint32)
        sdict = {f: getattr(stats, f) for f, _ in N.BatchStats._fields_}
        if not copy:
            return Results(qid, ent[:, :, 0], ent[:, :, 1], ln, thr, None, None, sdict)
        return Results(qid, ent[:, :, 0].copy(), ent[:, :, 1].copy(), ln, thr, None, None, sdict)


def _mcix_bytes(image) -> bytes:
    if isinstance(image, (bytes, bytearray, memoryview)):
        return bytes(image)
    with open(image, "rb") as f:
        return f.read()


def mcix_parse(image) -> CSR:
    """deserialize_index (index_io.hpp:84-146) as CSR, on the host (no GPU):
    the same validation and DataError messages as the reference."""
    data = _mcix_bytes(image)
    lib = N.engine()
    buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data or b"\0")
    n, K, P, err = C.c_uint32(), C.c_uint64(), C.c_uint64(), _errbuf()
    check(lib.genie_mcix_parse(C.cast(buf, C.c_void_p), len(data), C.byref(n), C.byref(K), C.byref(P), None, None,
                               None, err, len(err)), err)
    keys = np.zeros(K.value, np.uint64)
    off = np.zeros(K.value + 1, np.uint64)
    post = np.zeros(max(1, P.value), np.uint32)
    check(lib.genie_mcix_parse(C.cast(buf, C.c_void_p), len(data), None, None, None, _ptr(keys, C.c_uint64),
                               _ptr(off, C.c_uint64), _ptr(post, C.c_uint32), err, len(err)), err)
    return CSR(n.value, keys, off, post[:P.value])


def mcix_serialize(csr: CSR, split: Optional[int] = 4096) -> bytes:
    """serialize_index (index_io.hpp:63-82) of build_index(objects, split)
    (index.hpp:190-250) for the objects this CSR holds; split None = whole
    lists (the reference's default build)."""
    lib = N.engine()
    size, err = C.c_uint64(0), _errbuf()
    key_off = csr.key_off if csr.key_off.size else np.zeros(1, np.uint64)
    args = (csr.n, csr.num_keys, _ptr(csr.keys, C.c_uint64), _ptr(key_off, C.c_uint64),
            _ptr(csr.postings, C.c_uint32), 0 if split is None else int(split))
    check(lib.genie_mcix_serialize(*args, None, C.byref(size), err, len(err)), err)
    out = (C.c_uint8 * max(1, size.value))()
    check(lib.genie_mcix_serialize(*args, C.cast(out, C.c_void_p), C.byref(size), err, len(err)), err)
    return bytes(out)[: size.value]


def point_queries(tokens: np.ndarray, k: int, first_id: int = 0) -> QueryBatch:
    """encode_query_point (lsh.hpp:186-195) for a batch: query q has items
    (i, tokens[q, i]) for every function i."""
    Q, m = tokens.shape
    return QueryBatch(
        qid=np.arange(first_id, first_id + Q, dtype=np.uint32),
        k=np.full(Q, k, np.uint32),
        item_off=np.arange(Q + 1, dtype=np.uint64) * m,
        dim=np.tile(np.arange(m, dtype=np.uint16), Q),
        lo=tokens.reshape(-1).astype(np.uint32),
        hi=tokens.reshape(-1).astype(np.uint32),
    )


def csr_from_tokens(tokens: np.ndarray) -> CSR:
    """Host CSR for LSH tokens (dim = function index), ids ascending per key."""
    n, m = tokens.shape
    keys_all = (np.arange(m, dtype=np.uint64)[None, :] << np.uint64(32)) | tokens.astype(np.uint64)
    flat = keys_all.reshape(-1)
    order = np.argsort(flat, kind="stable")
    sk = flat[order]
    ids = (order // m).astype(np.uint32)
    uniq, starts = np.unique(sk, return_index=True)
    off = np.concatenate([starts.astype(np.uint64), np.array([sk.shape[0]], np.uint64)])
    return CSR(n, uniq, off, ids)


def kernel_width_heuristic(points: np.ndarray, max_pairs: int = 1_000_000) -> float:
    """Mean pairwise l1 distance (lsh.hpp:333-363), vectorised: all pairs when
    n(n-1)/2 <= max_pairs, else max_pairs pairs drawn with the reference's
    SplitMix64(0x6d63782d7730) sequence.  Summation order differs from the
    reference's sequential loop, so the last bits of sigma may differ; sigma is
    an explicit input of the encoder on every path that is compared."""
    pts = np.asarray(points, np.float64)
    n = pts.shape[0]
    if n < 2:
        raise ContractError("kernel width needs at least 2 points")
    total = n * (n - 1) // 2
    if total <= max_pairs:
        ii, jj = np.triu_indices(n, 1)
    else:
        gamma = np.uint64(0x9E3779B97F4A7C15)
        t = np.arange(1, 2 * max_pairs + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(0x6D63782D7730) + t * gamma
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        ii = (z[0::2] % np.uint64(n)).astype(np.int64)
        jj = (z[1::2] % np.uint64(n - 1)).astype(np.int64)
        jj += (jj >= ii)
    acc = 0.0
    for a in range(0, ii.shape[0], 65536):
        acc += float(np.abs(pts[ii[a:a + 65536]] - pts[jj[a:a + 65536]]).sum())
    return acc / ii.shape[0]
