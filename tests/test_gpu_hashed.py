"""The hashed sparse class of k_scan (k_scan<kHashW>, genie_query.cu): queries
whose postings are few for the objects they spread over count into a
shared-memory open-addressing table over tiles of GENIE_HASH_TILES x the
W = 8 tile, with the c-PQ threshold read off the final counts and a radix
selection of the tie ids.  By default it takes only queries with at most
GENIE_HASH_DENSE_MAX expected postings per W = 8 tile (ultra-sparse: there it
is 1.4-4.3x faster; at C4's ~1 500 the dense tiles win); these
tests also switch it on through its knobs for denser queries and compare every
case with the CPU oracle (cpq.hpp:307-339 extract semantics,
engine.hpp:158-177 merge), across knob values, which must not change results."""
import os

import numpy as np
import pytest

from paper_1603_08390_b200 import DeviceIndex, point_queries
from paper_1603_08390_b200.engine import CSR, QueryBatch

pytestmark = pytest.mark.gpu


def assert_same(got, want, label):
    assert np.array_equal(got.length, want.length), label
    assert np.array_equal(got.threshold, want.threshold), label
    for q in range(len(got.length)):
        assert got.row(q) == want.row(q), f"{label} q{q}"


# the class on for queries it would not take by default (C4-like density)
HASH_ON = {"GENIE_HASH_TILES": 4, "GENIE_HASH_DENSE_MAX": 1 << 20, "GENIE_HASH_MIN_ITEMS": 0, "GENIE_HASH_LAUNCH": 1}


class env:
    def __init__(self, **kv):
        self.kv = {k: str(v) for k, v in kv.items()}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update(self.kv)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def minhash_like(n, m, domain, queries, rng, lo=0, hi=None, near=True):
    """n objects x m functions; the objects [lo, hi) carry postings (skew
    when the range is narrow), the token of (object, function) uniform in
    [0, domain).  Queries copy a random live object's tokens and perturb half
    of them (near=True) or draw fresh ones, so counts range over 1..m with
    many ties at the low levels."""
    hi = n if hi is None else hi
    toks = rng.integers(0, domain, size=(hi - lo, m), dtype=np.uint32)
    flat = ((np.arange(m, dtype=np.uint64)[None, :] << np.uint64(32)) | toks.astype(np.uint64)).reshape(-1)
    ids = np.repeat(np.arange(lo, hi, dtype=np.uint32), m)
    order = np.argsort(flat, kind="stable")
    sk, sid = flat[order], ids[order]
    uniq, starts = np.unique(sk, return_index=True)
    off = np.concatenate([starts.astype(np.uint64), np.array([sk.shape[0]], np.uint64)])
    csr = CSR(n, uniq, off, sid)
    qt = toks[rng.integers(0, hi - lo, size=queries)].copy()
    if near:
        flip = rng.random(qt.shape) < 0.5
        qt[flip] = rng.integers(0, domain, size=int(flip.sum()), dtype=np.uint32)
    else:
        qt = rng.integers(0, domain, size=qt.shape, dtype=np.uint32)
    return csr, qt


@pytest.fixture(scope="module")
def multi_tile(gpu, oracle):
    rng = np.random.default_rng(11)
    csr, qt = minhash_like(900_000, 64, 4096, 96, rng)
    ix = DeviceIndex.from_csr(csr, device=gpu)
    qb = point_queries(qt, 100)
    want = oracle.index(csr).execute(qb)
    yield csr, ix, qb, want
    ix.close()


def test_hashed_multi_tile_equals_oracle(multi_tile):
    csr, ix, qb, want = multi_tile
    with env(**HASH_ON):
        got = ix.query(qb)
    assert_same(got, want, "hashed")
    # the class engaged (its minimum batch share waived): 3 hashed tiles per
    # query instead of 10 W = 8 tiles
    assert got.stats["work_items"] < len(qb) * 4
    assert got.stats["fallback_tiles"] == 0
    # by default this density (~1 500 postings per W = 8 tile) stays on dense tiles
    assert ix.query(qb).stats["work_items"] == len(qb) * 10


@pytest.mark.parametrize("knobs", [
    {"GENIE_HASH_TILES": 0},           # class off: W = 8 dense tiles
    {**HASH_ON, "GENIE_HASH_FILL_PCT": 0},  # every hashed item through the 8-bit sub-tile path
    {**HASH_ON, "GENIE_HASH_TILES": 1},  # hashed tiles of one W = 8 tile
    {**HASH_ON, "GENIE_HASH_TILES": 11, "GENIE_HASH_LOAD_PCT": 100, "GENIE_HASH_FILL_PCT": 90},  # 2^20 objects
    {**HASH_ON, "GENIE_HASH_LOAD_PCT": 5},  # admission threshold: a mix of classes
])
def test_hashed_knobs_are_result_invariant(multi_tile, knobs):
    csr, ix, qb, want = multi_tile
    with env(**knobs):
        got = ix.query(qb)
    assert_same(got, want, str(knobs))
    if knobs.get("GENIE_HASH_FILL_PCT") == 0:
        assert got.stats["fallback_tiles"] > 0


@pytest.mark.parametrize("k", [1, 7, 100, 1000, 5000])
def test_hashed_tie_selection(gpu, oracle, k):
    # unrelated queries: almost every count is 1 or 2, so the k-th count has
    # thousands of ties and the radix cut on the tie ids decides the rows
    rng = np.random.default_rng(k)
    csr, qt = minhash_like(700_000, 32, 2048, 24, rng, near=False)
    qb = point_queries(qt, k)
    ix = DeviceIndex.from_csr(csr, device=gpu)
    with env(**HASH_ON):
        got = ix.query(qb)
    want = oracle.index(csr).execute(qb)
    assert_same(got, want, f"k={k}")
    ix.close()


def test_hashed_skewed_tile_takes_sub_tile_path(gpu, oracle):
    # every posting in the first 60K ids of 3M objects: the query's expected
    # postings per hashed tile are small, its first tile holds all of them
    rng = np.random.default_rng(5)
    csr, qt = minhash_like(3_000_000, 128, 512, 16, rng, lo=0, hi=60_000)
    qb = point_queries(qt, 100)
    ix = DeviceIndex.from_csr(csr, device=gpu)
    with env(**HASH_ON):
        got = ix.query(qb)
    want = oracle.index(csr).execute(qb)
    assert_same(got, want, "skewed")
    assert got.stats["fallback_tiles"] > 0
    ix.close()


def test_hashed_ranges_and_gate_floors(gpu, oracle):
    # range items (several keywords per item) and mixed k per query
    rng = np.random.default_rng(9)
    csr, qt = minhash_like(800_000, 32, 1 << 14, 40, rng)
    Q, m = qt.shape
    width = rng.integers(0, 3, size=(Q, m)).astype(np.uint32)
    lo = qt.reshape(-1)
    hi = np.minimum(lo + width.reshape(-1), (1 << 14) - 1).astype(np.uint32)
    qb = QueryBatch(qid=np.arange(Q, dtype=np.uint32), k=rng.integers(1, 300, size=Q).astype(np.uint32),
                    item_off=np.arange(Q + 1, dtype=np.uint64) * m, dim=np.tile(np.arange(m, dtype=np.uint16), Q),
                    lo=lo, hi=hi)
    ix = DeviceIndex.from_csr(csr, device=gpu)
    with env(**HASH_ON):
        got = ix.query(qb)
    want = oracle.index(csr).execute(qb)
    assert_same(got, want, "ranges")
    ix.close()


def sparse_sets(n, live, m, domain, queries, rng):
    """`live` objects spread over n ids (ultra-sparse lists)."""
    ids = np.sort(rng.choice(n, size=live, replace=False)).astype(np.uint32)
    toks = rng.integers(0, domain, size=(live, m), dtype=np.uint32)
    flat = ((np.arange(m, dtype=np.uint64)[None, :] << np.uint64(32)) | toks.astype(np.uint64)).reshape(-1)
    oid = np.repeat(ids, m)
    order = np.argsort(flat, kind="stable")
    sk, sid = flat[order], oid[order]
    uniq, starts = np.unique(sk, return_index=True)
    off = np.concatenate([starts.astype(np.uint64), np.array([sk.shape[0]], np.uint64)])
    qt = toks[rng.integers(0, live, size=queries)].copy()
    flip = rng.random(qt.shape) < 0.5
    qt[flip] = rng.integers(0, domain, size=int(flip.sum()), dtype=np.uint32)
    return CSR(n, uniq, off, sid), qt


def test_hashed_class_by_default_on_ultra_sparse(gpu, oracle):
    # 400K sets over 12M ids: ~65 postings per W = 8 tile -> hashed 2^20-object
    # tiles by default (12 per query instead of 126 dense tiles)
    rng = np.random.default_rng(21)
    csr, qt = sparse_sets(12_000_000, 400_000, 32, 2048, 64, rng)
    qb = point_queries(qt, 100)
    ix = DeviceIndex.from_csr(csr, device=gpu)
    want = oracle.index(csr).execute(qb)
    # the first batch on the index runs dense tiles and flags the class; the
    # class's kernel is launched from the next batch on
    first = ix.query(qb)
    assert first.stats["work_items"] == len(qb) * 126
    assert_same(first, want, "ultra-sparse, first batch")
    got = ix.query(qb)
    assert got.stats["work_items"] == len(qb) * 12
    assert_same(got, want, "ultra-sparse")
    with env(GENIE_HASH_TILES=0):
        dense = ix.query(qb)
    assert dense.stats["work_items"] == len(qb) * 126
    assert_same(dense, want, "ultra-sparse dense tiles")
    # a few such queries in a batch (fewer hashed items than two per scan CTA)
    # go back to dense tiles instead of a separate, mostly idle launch
    few = qb.slice(0, 8)
    got_few = ix.query(few)
    assert got_few.stats["work_items"] == len(few) * 126
    assert_same(got_few, oracle.index(csr).execute(few), "few ultra-sparse")
    ix.close()
