"""Seeded synthetic workloads of the BASELINE.json configs,
generated natively (libgenie_synth.so).  Input preparation only.

C1 adult    48 842 x 14 relational rows, 1024 queries, k=100
C2 tweets   7M docs, vocab 1M, 10 Zipf(1) words, 1024 queries, k=100
C3 sift     4M x 128-d mixture, 1024 queries (E2LSH m=237 -> match count)
C4 minhash  2M sets, 128 functions, 4096 queries, k=100
C5 ocr      1M x 784-d in [0,1], 2048 queries, k=1 (1-NN prediction)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N
from .engine import CSR, QueryBatch

SEEDS = {"adult": 0xAD017, "tweets": 12345, "sift": 0x51F7, "minhash": 0x4D494E48, "ocr": 0x4F4352}


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


@dataclass
class Dataset:
    csr: Optional[CSR] = None
    queries: Optional[QueryBatch] = None
    points: Optional[np.ndarray] = None
    query_points: Optional[np.ndarray] = None
    labels: Optional[np.ndarray] = None
    query_labels: Optional[np.ndarray] = None
    set_off: Optional[np.ndarray] = None
    elems: Optional[np.ndarray] = None
    query_set_off: Optional[np.ndarray] = None
    query_elems: Optional[np.ndarray] = None


def _collect(h: C.c_void_p) -> Dataset:
    lib = N.synth()
    ds = Dataset()
    n, K = C.c_uint32(), C.c_uint64()
    keys, off, post = N.u64p(), N.u64p(), N.u32p()
    lib.genie_dataset_csr(h, C.byref(n), C.byref(K), C.byref(keys), C.byref(off), C.byref(post))
    if K.value or n.value:
        nk = K.value
        key_off = _arr(off, nk + 1, np.uint64)
        ds.csr = CSR(n.value, _arr(keys, nk, np.uint64), key_off, _arr(post, int(key_off[-1]) if nk else 0, np.uint32))
    Q = C.c_uint32()
    qid, kk, ioff, dim, lo, hi = N.u32p(), N.u32p(), N.u64p(), N.u16p(), N.u32p(), N.u32p()
    lib.genie_dataset_queries(h, C.byref(Q), C.byref(qid), C.byref(kk), C.byref(ioff), C.byref(dim), C.byref(lo),
                              C.byref(hi))
    if Q.value:
        item_off = _arr(ioff, Q.value + 1, np.uint64)
        ni = int(item_off[-1])
        ds.queries = QueryBatch(_arr(qid, Q.value, np.uint32), _arr(kk, Q.value, np.uint32), item_off,
                                _arr(dim, ni, np.uint16), _arr(lo, ni, np.uint32), _arr(hi, ni, np.uint32))
    pn, dims, pq = C.c_uint32(), C.c_uint32(), C.c_uint32()
    pts, qpts, lab, qlab = N.f32p(), N.f32p(), N.u32p(), N.u32p()
    lib.genie_dataset_points(h, C.byref(pn), C.byref(dims), C.byref(pts), C.byref(pq), C.byref(qpts), C.byref(lab),
                             C.byref(qlab))
    if pn.value:
        ds.points = _arr(pts, pn.value * dims.value, np.float32).reshape(pn.value, dims.value)
        ds.query_points = _arr(qpts, pq.value * dims.value, np.float32).reshape(pq.value, dims.value)
        if lab:
            try:
                ds.labels = _arr(lab, pn.value, np.uint32)
                ds.query_labels = _arr(qlab, pq.value, np.uint32)
            except ValueError:
                pass
    sn, sq = C.c_uint32(), C.c_uint32()
    soff, sel, qoff, qel = N.u64p(), N.u64p(), N.u64p(), N.u64p()
    lib.genie_dataset_sets(h, C.byref(sn), C.byref(soff), C.byref(sel), C.byref(sq), C.byref(qoff), C.byref(qel))
    if sn.value:
        ds.set_off = _arr(soff, sn.value + 1, np.uint64)
        ds.elems = _arr(sel, int(ds.set_off[-1]), np.uint64)
        ds.query_set_off = _arr(qoff, sq.value + 1, np.uint64)
        ds.query_elems = _arr(qel, int(ds.query_set_off[-1]), np.uint64)
    lib.genie_dataset_free(h)
    return ds


def _make(fn, *args) -> Dataset:
    h = C.c_void_p()
    rc = fn(*args, C.byref(h))
    if rc != 0:
        raise ValueError(f"synthetic generator failed ({rc})")
    return _collect(h)


def adult(n: int = 48842, queries: int = 1024, k: int = 100, seed: int = SEEDS["adult"]) -> Dataset:
    return _make(N.synth().genie_synth_adult, n, queries, k, seed)


def tweets(n: int = 7_000_000, vocab: int = 1_000_000, words: int = 10, queries: int = 1024, k: int = 100,
           seed: int = SEEDS["tweets"]) -> Dataset:
    return _make(N.synth().genie_synth_tweets, n, vocab, words, queries, k, seed)


def sift(n: int = 4_000_000, dims: int = 128, queries: int = 1024, seed: int = SEEDS["sift"]) -> Dataset:
    return _make(N.synth().genie_synth_sift, n, dims, queries, seed)


def ocr(n: int = 1_000_000, dims: int = 784, queries: int = 2048, seed: int = SEEDS["ocr"]) -> Dataset:
    return _make(N.synth().genie_synth_ocr, n, dims, queries, seed)


def sets(n: int = 2_000_000, queries: int = 4096, seed: int = SEEDS["minhash"]) -> Dataset:
    return _make(N.synth().genie_synth_sets, n, queries, seed)


def random_instance(n: int, dims: int = 4, tokens: int = 8, max_kw: int = 5, queries: int = 8, max_items: int = 4,
                    max_span: int = 2, max_k: int = 10, seed: int = 1) -> Dataset:
    """Small random instance shaped like test_engine.cpp:34-60."""
    return _make(N.synth().genie_synth_random, n, dims, tokens, max_kw, queries, max_items, max_span, max_k, seed)


def csr_from_objects(n: int, obj_off: np.ndarray, dims: np.ndarray, tokens: np.ndarray) -> CSR:
    obj_off = np.ascontiguousarray(obj_off, np.uint64)
    dims = np.ascontiguousarray(dims, np.uint16)
    tokens = np.ascontiguousarray(tokens, np.uint32)
    h, err = C.c_void_p(), C.create_string_buffer(512)
    rc = N.synth().genie_synth_csr_from_objects(n, obj_off.ctypes.data_as(N.u64p), dims.ctypes.data_as(N.u16p),
                                                tokens.ctypes.data_as(N.u32p), C.byref(h), err, len(err))
    if rc == 1:
        from .engine import ContractError
        raise ContractError(err.value.decode())
    if rc:
        raise ValueError(err.value.decode())
    ds = _collect(h)
    return ds.csr if ds.csr is not None else CSR(n, np.zeros(0, np.uint64), np.zeros(1, np.uint64),
                                                 np.zeros(0, np.uint32))
