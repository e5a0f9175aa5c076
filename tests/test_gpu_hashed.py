"""The hashed sparse class of k_scan (k_scan<kHashW>, genie_query.cu): queries
whose postings are few for the objects they spread over count into a
shared-memory open-addressing table over tiles of GENIE_HASH_TILES x the
W = 8 tile, with the c-PQ threshold read off the final counts and a radix
selection of the tie ids.  The class is off by default (measured slower than
the dense W = 8 tiles on C4); these tests switch it on through
its knobs and compare every case with the CPU oracle (cpq.hpp:307-339 extract
semantics, engine.hpp:158-177 merge), across knob values, which must not
change results."""
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


HASH_ON = {"GENIE_HASH_TILES": 4}


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
    # the class engaged: 3 hashed tiles per query instead of 10 W = 8 tiles
    assert got.stats["work_items"] < len(qb) * 4
    assert got.stats["fallback_tiles"] == 0
    # off by default
    assert ix.query(qb).stats["work_items"] == len(qb) * 10


@pytest.mark.parametrize("knobs", [
    {"GENIE_HASH_TILES": 0},           # class off (the default): W = 8 dense tiles
    {"GENIE_HASH_TILES": 4, "GENIE_HASH_FILL_PCT": 0},  # every hashed item through the 8-bit sub-tile path
    {"GENIE_HASH_TILES": 1},           # hashed tiles of one W = 8 tile
    {"GENIE_HASH_TILES": 9, "GENIE_HASH_LOAD_PCT": 100, "GENIE_HASH_FILL_PCT": 90},  # 2^20-object tile cap
    {"GENIE_HASH_TILES": 4, "GENIE_HASH_LOAD_PCT": 5},  # admission threshold: a mix of classes
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
