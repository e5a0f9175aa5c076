"""Object-level mirror of the reference API (namespace mcx, /root/reference/proj/include).

Same names, argument meaning and error behaviour as the reference headers,
with the batched query path executed by the sm_100a engine through the C ABI.
Host-side pieces that the reference also runs on the host (object/query
construction, build_index's CSR, partition bookkeeping, merge_topk,
hash_results) are restated here; match counting and top-k selection run on
the GPU.  File:line citations refer to /root/reference/proj/include/mcx/.
"""
from __future__ import annotations

import enum
import time
from dataclasses import dataclass, field
from typing import Iterable, List, NamedTuple, Optional, Sequence

import numpy as np

from . import engine as E
from .engine import ContractError, DataError, InvariantError  # noqa: F401  (error.hpp:24-41)

DimId = int
Token = int
ObjectId = int

# ------------------------------------------------------------------ model.hpp


class Keyword(NamedTuple):
    """(dimension, token) universe element (model.hpp:36-46)."""

    dim: int
    token: int

    def packed(self) -> int:
        return (int(self.dim) << 32) | int(self.token)


class ObjectRecord:
    """Sorted, duplicate-free keyword set (model.hpp:52-71)."""

    __slots__ = ("_id", "_keywords")

    def __init__(self, id: int, keywords: Iterable):
        kws = sorted(Keyword(int(k[0]), int(k[1])) for k in keywords)
        for a, b in zip(kws, kws[1:]):
            if a == b:
                raise ContractError(f"ObjectRecord {id}: duplicate keyword (dim={a.dim}, token={a.token})")
        self._id = int(id)
        self._keywords = kws

    def id(self) -> int:
        return self._id

    def keywords(self) -> List[Keyword]:
        return self._keywords


class QueryItem:
    """Inclusive token range on one dimension (model.hpp:74-88)."""

    __slots__ = ("dim", "lo", "hi")

    def __init__(self, dim: int, lo: int, hi: int):
        if lo > hi:
            raise ContractError(f"QueryItem: lo {lo} > hi {hi} on dim {dim}")
        self.dim, self.lo, self.hi = int(dim), int(lo), int(hi)

    @staticmethod
    def point(dim: int, token: int) -> "QueryItem":
        return QueryItem(dim, token, token)

    def __repr__(self):
        return f"QueryItem({self.dim}, {self.lo}, {self.hi})"


class Query:
    """Range-item query asking for the k best objects (model.hpp:91-102)."""

    __slots__ = ("id", "items", "k")

    def __init__(self, id: int, items: Sequence[QueryItem], k: int):
        items = list(items)
        if not items:
            raise ContractError(f"Query {id}: no items")
        if k == 0:
            raise ContractError(f"Query {id}: k must be >= 1")
        self.id, self.items, self.k = int(id), items, int(k)


def match_count_reference(query: Query, obj: ObjectRecord) -> int:
    """The semantic definition of a match count (model.hpp:107-116)."""
    import bisect

    kws = obj.keywords()
    total = 0
    for it in query.items:
        a = bisect.bisect_left(kws, Keyword(it.dim, it.lo))
        b = bisect.bisect_right(kws, Keyword(it.dim, it.hi))
        total += b - a
    return total


class RelationalSchema:
    """Per-attribute token domains (model.hpp:119-137)."""

    def __init__(self, domain_sizes: Sequence[int]):
        if not domain_sizes:
            raise ContractError("RelationalSchema: empty schema")
        for a, d in enumerate(domain_sizes):
            if d == 0:
                raise ContractError(f"RelationalSchema: attribute {a} has empty domain")
        self._d = [int(x) for x in domain_sizes]

    def attribute_count(self) -> int:
        return len(self._d)

    def domain_size(self, attr: int) -> int:
        return self._d[attr]


def encode_relational_tuple(schema: RelationalSchema, values: Sequence[int], id: int) -> ObjectRecord:
    """model.hpp:140-157"""
    if len(values) != schema.attribute_count():
        raise ContractError(f"tuple arity {len(values)} != schema arity {schema.attribute_count()}")
    kws = []
    for a, v in enumerate(values):
        if v >= schema.domain_size(a):
            raise DataError(f"attribute {a}: token {v} outside domain [0, {schema.domain_size(a)})")
        kws.append(Keyword(a, int(v)))
    return ObjectRecord(id, kws)


@dataclass
class AttributeRange:
    attr: int = 0
    lo: int = 0
    hi: int = 0


def encode_relational_query(schema: RelationalSchema, ranges: Sequence[AttributeRange], k: int,
                            query_id: int = 0) -> Query:
    """Ranges clamped into the attribute domains (model.hpp:167-188)."""
    items = []
    for r in ranges:
        if r.attr >= schema.attribute_count():
            raise ContractError(f"range on unknown attribute {r.attr}")
        dom = schema.domain_size(r.attr)
        lo, hi = max(r.lo, 0), min(r.hi, dom - 1)
        if lo > hi:
            raise DataError(f"attribute {r.attr}: range [{r.lo}, {r.hi}] is empty after clamping to [0, {dom})")
        items.append(QueryItem(r.attr, lo, hi))
    return Query(query_id, items, k)


# --------------------------------------------------------------------- sa.hpp


def tokenize_document(text: str, stop_words: Iterable[str] = ()) -> List[str]:
    """Lowercased whitespace-separated words minus stop words, deduplicated and
    sorted (tokenize_document, sa.hpp:341-359).  Whitespace and lowercasing are
    the C locale's (ASCII), as std::isspace / std::tolower there."""
    stop = set(stop_words)
    words = set()
    cur: List[str] = []

    def flush():
        if cur:
            w = "".join(cur)
            if w not in stop:
                words.add(w)
            cur.clear()

    for ch in text:
        if ch in " \t\n\v\f\r":
            flush()
        else:
            cur.append(ch.lower() if "A" <= ch <= "Z" else ch)
    flush()
    return sorted(words)


class DocumentCodec:
    """Word vocabulary for bag-of-words documents (DocumentCodec, sa.hpp:361-408):
    token = the word's rank in the sorted build-corpus vocabulary, all on dim 0,
    so the match count of two encoded documents is the size of their word-set
    intersection (the Tweets workload)."""

    def __init__(self):
        self._stop: set = set()
        self._vocab: dict = {}

    @staticmethod
    def build(corpus: Iterable[str], stop_words: Iterable[str] = ()) -> "DocumentCodec":
        c = DocumentCodec()
        c._stop = set(stop_words)
        words = set()
        for doc in corpus:
            words.update(tokenize_document(doc, c._stop))
        c._vocab = {w: i for i, w in enumerate(sorted(words))}
        return c

    def vocabulary_size(self) -> int:
        return len(self._vocab)

    def encode(self, text: str, id: int) -> ObjectRecord:
        kws = []
        for w in tokenize_document(text, self._stop):
            if w not in self._vocab:
                raise ContractError("document word outside the vocabulary")
            kws.append(Keyword(0, self._vocab[w]))
        return ObjectRecord(id, kws)

    def encode_query(self, text: str, k: int, query_id: int = 0) -> Optional[Query]:
        """Words outside the vocabulary are dropped; None when nothing is left."""
        items = [QueryItem.point(0, self._vocab[w]) for w in tokenize_document(text, self._stop) if w in self._vocab]
        return Query(query_id, items, k) if items else None


# -------------------------------------------------------------------- cpq.hpp


class TopKEntry(NamedTuple):
    id: int
    count: int

    @staticmethod
    def better(a: "TopKEntry", b: "TopKEntry") -> bool:
        """count desc, id asc (cpq.hpp:37-40)"""
        if a.count != b.count:
            return a.count > b.count
        return a.id < b.id


def _order_key(e: TopKEntry):
    return (-e.count, e.id)


@dataclass
class TopKResult:
    query_id: int = 0
    entries: List[TopKEntry] = field(default_factory=list)  # count desc, id asc
    threshold: int = 0


def width_for(max_count: int) -> int:
    """cpq.hpp:63-68"""
    for w in (4, 8, 16):
        if max_count <= (1 << w) - 1:
            return w
    return 32


# ------------------------------------------------------------------ index.hpp

kDefaultSplitThreshold = 4096


class PostingsSpan(NamedTuple):
    begin: int
    end: int

    def length(self) -> int:
        return self.end - self.begin


@dataclass
class KeywordEntry:
    keyword: Keyword
    first_span: int
    span_count: int


class InvertedIndex:
    """Position map + one postings array (index.hpp:41-182).  The host keeps
    the CSR; the device copy (DeviceIndex) is created on first query."""

    def __init__(self, csr: E.CSR, split_threshold: Optional[int] = None, device: int = 0):
        self.csr = csr
        self._split = split_threshold
        self._device = device
        self._dev: Optional[E.DeviceIndex] = None
        self._dim_mult: Optional[np.ndarray] = None

    # accessors (index.hpp:68-81)
    def num_objects(self) -> int:
        return int(self.csr.n)

    def keyword_count(self) -> int:
        return self.csr.num_keys

    def list_array(self) -> np.ndarray:
        return self.csr.postings

    def split_threshold(self) -> Optional[int]:
        return self._split

    def _spans_of_key(self, j: int) -> List[PostingsSpan]:
        b, e = int(self.csr.key_off[j]), int(self.csr.key_off[j + 1])
        if not self._split:
            return [PostingsSpan(b, e)]
        return [PostingsSpan(p, min(p + self._split, e)) for p in range(b, e, self._split)]

    def entries(self) -> List[KeywordEntry]:
        out, first = [], 0
        for j, key in enumerate(self.csr.keys.tolist()):
            cnt = len(self._spans_of_key(j))
            out.append(KeywordEntry(Keyword(key >> 32, key & 0xFFFFFFFF), first, cnt))
            first += cnt
        return out

    def spans(self) -> List[PostingsSpan]:
        return [s for j in range(self.csr.num_keys) for s in self._spans_of_key(j)]

    def ids(self, span: PostingsSpan) -> np.ndarray:
        return self.csr.postings[span.begin:span.end]

    def lookup(self, item: QueryItem) -> List[PostingsSpan]:
        """index.hpp:86-102"""
        keys = self.csr.keys
        a = int(np.searchsorted(keys, np.uint64((item.dim << 32) | item.lo), "left"))
        b = int(np.searchsorted(keys, np.uint64((item.dim << 32) | item.hi), "right"))
        return [s for j in range(a, b) for s in self._spans_of_key(j)]

    def _dim_stats(self) -> np.ndarray:
        if self._dim_mult is None:
            self._dim_mult = dim_stats(self.csr)
        return self._dim_mult

    def max_token(self, dim: int) -> Optional[int]:
        keys = self.csr.keys
        hi = int(np.searchsorted(keys, np.uint64(((dim + 1) << 32)), "left"))
        if hi == 0 or int(keys[hi - 1]) >> 32 != dim:
            return None
        return int(keys[hi - 1]) & 0xFFFFFFFF

    def max_multiplicity(self, dim: int) -> int:
        return int(self._dim_stats()[dim])

    def max_count_bound(self, query: Query) -> int:
        """index.hpp:118-133"""
        keys = self.csr.keys
        bound = 0
        for it in query.items:
            a = int(np.searchsorted(keys, np.uint64((it.dim << 32) | it.lo), "left"))
            b = int(np.searchsorted(keys, np.uint64((it.dim << 32) | it.hi), "right"))
            bound += min(b - a, self.max_multiplicity(it.dim))
        return bound

    def longest_list(self) -> int:
        return int(np.max(np.diff(self.csr.key_off))) if self.csr.num_keys else 0

    def device(self) -> E.DeviceIndex:
        if self._dev is None:
            self._dev = E.DeviceIndex.from_csr(self.csr, device=self._device, dim_max_mult=self._dim_stats())
        return self._dev


def dim_stats(csr: E.CSR) -> np.ndarray:
    """max_multiplicity per dim (index.hpp:153-174) on the host."""
    out = np.zeros(65536, np.uint32)
    if csr.num_keys == 0:
        return out
    dims = (csr.keys >> np.uint64(32)).astype(np.int64)
    lens = np.diff(csr.key_off).astype(np.int64)
    post_dim = np.repeat(dims, lens)
    for d in np.unique(dims):
        ids = csr.postings[post_dim == d]
        if ids.size:
            out[d] = np.bincount(ids).max()
    return out


def build_index(objects: Sequence[ObjectRecord], split_threshold: Optional[int] = None,
                device: int = 0) -> InvertedIndex:
    """index.hpp:190-250: dense ids 0..n-1 (any order), lists ascending."""
    if split_threshold is not None and split_threshold == 0:
        raise ContractError("split_threshold must be positive")
    n = len(objects)
    seen = np.zeros(n, bool)
    order = [None] * n
    for obj in objects:
        i = obj.id()
        if i >= n or seen[i]:
            raise DataError(f"object ids must be dense 0..{n - 1 if n else 0}: bad id {i}")
        seen[i] = True
        order[i] = obj
    from . import synth

    off = np.zeros(n + 1, np.uint64)
    dims, toks = [], []
    for i, obj in enumerate(order):
        kws = obj.keywords()
        off[i + 1] = off[i] + len(kws)
        dims.extend(k.dim for k in kws)
        toks.extend(k.token for k in kws)
    csr = synth.csr_from_objects(n, off, np.array(dims, np.uint16), np.array(toks, np.uint32))
    return InvertedIndex(csr, split_threshold, device)


# ---------------------------------------------------------------- index_io.hpp
# MCIX files (index_io.hpp:27-154): the reference's bytes for the same build,
# its validation and DataError messages on load.  A loaded index keeps
# whole-list spans (the file's span cut is a build-time choice).


def serialize_index(index: InvertedIndex) -> bytes:
    return E.mcix_serialize(index.csr, index.split_threshold())


def deserialize_index(data: bytes, device: int = 0) -> InvertedIndex:
    return InvertedIndex(E.mcix_parse(data), None, device)


def save_index(index: InvertedIndex, path: str) -> None:
    with open(path, "wb") as f:
        f.write(serialize_index(index))


def load_index(path: str, device: int = 0) -> InvertedIndex:
    with open(path, "rb") as f:
        return deserialize_index(f.read(), device)


@dataclass
class IndexPartition:
    """index.hpp:254-259"""

    part_id: int
    id_offset: int
    size: int
    index: InvertedIndex


def partition_dataset(objects: Sequence[ObjectRecord], part_capacity: int,
                      split_threshold: Optional[int] = None, device: int = 0) -> List[IndexPartition]:
    """index.hpp:263-291"""
    if part_capacity == 0:
        raise ContractError("part_capacity must be >= 1")
    for i, o in enumerate(objects):
        if o.id() != i:
            raise DataError("partitioning requires objects in dense id order")
    parts, start, pid = [], 0, 0
    while start < len(objects):
        cnt = min(part_capacity, len(objects) - start)
        local = [ObjectRecord(i, objects[start + i].keywords()) for i in range(cnt)]
        parts.append(IndexPartition(pid, start, cnt, build_index(local, split_threshold, device)))
        pid += 1
        start += cnt
    return parts


# ----------------------------------------------------------------- engine.hpp


class Selector(enum.IntEnum):
    cpq = 0
    bucket = 1
    sort = 2


class ExecMode(enum.IntEnum):
    parallel = 0
    sequential = 1


@dataclass
class EngineConfig:
    """engine.hpp:36-42.  Every knob is result-invariant; the device
    additionally takes tile_bytes / ctas_per_sm (0 = library default)."""

    selector: Selector = Selector.cpq
    mode: ExecMode = ExecMode.parallel
    workers: int = 0
    span_chunk: int = 4096
    max_spans_per_task: int = 2
    tile_bytes: int = 0
    ctas_per_sm: int = 0


@dataclass
class StageTimings:
    lookup_ns: int = 0
    match_ns: int = 0
    select_ns: int = 0
    merge_ns: int = 0
    total_ns: int = 0


@dataclass
class MemoryStats:
    counter_bytes: int = 0
    gate_bytes: int = 0
    table_bytes: int = 0


@dataclass
class BatchResult:
    results: List[TopKResult] = field(default_factory=list)
    timings: StageTimings = field(default_factory=StageTimings)
    memory: MemoryStats = field(default_factory=MemoryStats)


def hash_results(results: Sequence[TopKResult]) -> int:
    """engine.hpp:141-153"""
    from .engine import hash_results as _h

    Q = len(results)
    stride = max([len(r.entries) for r in results] + [1])
    ids = np.zeros((Q, stride), np.uint32)
    counts = np.zeros((Q, stride), np.uint32)
    for q, r in enumerate(results):
        for e, ent in enumerate(r.entries):
            ids[q, e], counts[q, e] = ent.id, ent.count
    return _h(np.array([r.query_id for r in results], np.uint32), np.array([r.threshold for r in results], np.uint32),
              np.array([len(r.entries) for r in results], np.uint32), ids, counts)


def merge_topk(locals_: Sequence[TopKResult], k: int, query_id: int) -> TopKResult:
    """engine.hpp:158-177: disjoint parts' lists (global ids) -> merged top-k."""
    entries = [e for loc in locals_ for e in loc.entries]
    ids = sorted(e.id for e in entries)
    for a, b in zip(ids, ids[1:]):
        if a == b:
            raise ContractError(f"merge_topk: object {a} reported by more than one partition")
    entries.sort(key=_order_key)
    entries = entries[:k]
    return TopKResult(query_id, entries, entries[-1].count if len(entries) >= k else 0)


def _to_batch(queries: Sequence[Query]) -> E.QueryBatch:
    Q = len(queries)
    off = np.zeros(Q + 1, np.uint64)
    dims, lo, hi = [], [], []
    for q, qu in enumerate(queries):
        off[q + 1] = off[q] + len(qu.items)
        for it in qu.items:
            dims.append(it.dim)
            lo.append(it.lo)
            hi.append(it.hi)
    return E.QueryBatch(np.array([q.id for q in queries], np.uint32), np.array([q.k for q in queries], np.uint32), off,
                        np.array(dims, np.uint16), np.array(lo, np.uint32), np.array(hi, np.uint32))


def _device_config(config: EngineConfig):
    if config.span_chunk == 0 or config.max_spans_per_task == 0:
        raise ContractError("span_chunk and max_spans_per_task must be positive")
    return E.config(selector=int(config.selector), span_chunk=int(config.span_chunk),
                    max_spans_per_task=int(config.max_spans_per_task), tile_bytes=int(config.tile_bytes),
                    ctas_per_sm=int(config.ctas_per_sm))


def _results_from(res: E.Results) -> List[TopKResult]:
    out = []
    for q in range(len(res.length)):
        n = int(res.length[q])
        out.append(TopKResult(int(res.qid[q]),
                              [TopKEntry(int(i), int(c)) for i, c in zip(res.ids[q, :n], res.counts[q, :n])],
                              int(res.threshold[q])))
    return out


def execute_batch(index: InvertedIndex, queries: Sequence[Query], config: EngineConfig = EngineConfig()) -> BatchResult:
    """engine.hpp:184-304 on the GPU: results in request order."""
    cfg = _device_config(config)
    t0 = time.perf_counter_ns()
    batch = BatchResult()
    if not queries:
        batch.timings.total_ns = time.perf_counter_ns() - t0
        return batch
    qb = _to_batch(queries)
    res = index.device().query(qb, cfg, timings=True)
    batch.results = _results_from(res)
    t = res.timings
    batch.timings = StageTimings(t["lookup_ns"], t["match_ns"], t["select_ns"], t["merge_ns"],
                                 max(t["total_ns"], time.perf_counter_ns() - t0))
    s = res.stats
    batch.memory = MemoryStats(s["counter_bytes"], s["gate_bytes"], s["table_bytes"])
    return batch


def execute_partitioned(partitions: Sequence[IndexPartition], queries: Sequence[Query],
                        config: EngineConfig = EngineConfig()) -> BatchResult:
    """engine.hpp:308-347: each part on the GPU, then merge_topk (engine.hpp:158-177)."""
    expected = 0
    for part in partitions:
        if part.id_offset != expected or part.index.num_objects() != part.size:
            raise ContractError("partitions must be disjoint and contiguous")
        expected += part.size
    t0 = time.perf_counter_ns()
    batch = BatchResult(results=[TopKResult() for _ in queries])
    locals_ = [[] for _ in queries]
    for part in partitions:
        local = execute_batch(part.index, queries, config)
        batch.timings.lookup_ns += local.timings.lookup_ns
        batch.timings.match_ns += local.timings.match_ns
        batch.timings.select_ns += local.timings.select_ns
        batch.memory.counter_bytes = max(batch.memory.counter_bytes, local.memory.counter_bytes)
        batch.memory.gate_bytes = max(batch.memory.gate_bytes, local.memory.gate_bytes)
        batch.memory.table_bytes = max(batch.memory.table_bytes, local.memory.table_bytes)
        for q, r in enumerate(local.results):
            locals_[q].append(TopKResult(r.query_id, [TopKEntry(e.id + part.id_offset, e.count) for e in r.entries],
                                         r.threshold))
    t1 = time.perf_counter_ns()
    for q, qu in enumerate(queries):
        batch.results[q] = merge_topk(locals_[q], qu.k, qu.id)
    batch.timings.merge_ns = time.perf_counter_ns() - t1
    batch.timings.total_ns = time.perf_counter_ns() - t0
    return batch


# -------------------------------------------------------------------- lsh.hpp


class LshFamily(enum.IntEnum):
    p_stable = 0
    random_binning = 1
    min_hash = 2  # new; not in the reference


@dataclass
class LshEncoderConfig:
    """lsh.hpp:132-145 defaults."""

    family: LshFamily = LshFamily.random_binning
    m: int = 237
    dims: int = 0
    seed: int = 1
    rehash_domain: int = 8192
    w: float = 4.0
    bucket_count: int = 67
    bucket_min: int = -33
    rehash_pstable: bool = False
    sigma: float = 1.0


class LshEncoder:
    """lsh.hpp:149-219 with the transforms on the GPU (bit-exact fp64)."""

    def __init__(self, config: LshEncoderConfig, device: int = 0):
        self._cfg = config
        self._enc = E.Encoder(E.lsh_config(int(config.family), config.m, config.dims, config.seed,
                                           config.rehash_domain, config.w, config.bucket_count, config.bucket_min,
                                           config.rehash_pstable, config.sigma), device)

    @staticmethod
    def create(config: LshEncoderConfig, device: int = 0) -> "LshEncoder":
        return LshEncoder(config, device)

    def config(self) -> LshEncoderConfig:
        return self._cfg

    def m(self) -> int:
        return self._cfg.m

    def tokens(self, points: np.ndarray) -> np.ndarray:
        pts = np.asarray(points, np.float32)
        if pts.ndim == 1:
            pts = pts[None, :]
        if pts.shape[1] != self._cfg.dims:
            raise ContractError(f"point dimensionality {pts.shape[1]} != hash dimensionality {self._cfg.dims}")
        return self._enc.encode(pts)

    def token(self, function: int, point) -> int:
        if function >= self._cfg.m:
            raise ContractError("hash function index out of range")
        return int(self.tokens(point)[0, function])

    def encode_point(self, point, id: int) -> ObjectRecord:
        t = self.tokens(point)[0]
        return ObjectRecord(id, [Keyword(i, int(x)) for i, x in enumerate(t)])

    def encode_query_point(self, point, k: int, query_id: int = 0) -> Query:
        t = self.tokens(point)[0]
        return Query(query_id, [QueryItem.point(i, int(x)) for i, x in enumerate(t)], k)
