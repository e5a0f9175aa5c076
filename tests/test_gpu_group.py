"""Device groups (genie_group_*): one host thread drives
object-id-range shards, exchanges the per-shard top-k rows and merges them on
the first device.  On the single-GPU test box every shard sits on cuda:0 (the
peer-copy exchange, shards running concurrently on their own streams); a
one-shard group exercises the NCCL all-gather path.  Results must equal the
whole-index batch (execute_partitioned == execute_batch, acceptance.cpp:540-559)
and the CPU oracle."""
import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_1603_08390_b200 import DeviceGroup, DeviceIndex, _native as N, hash_results, synth
from paper_1603_08390_b200.dist import shard_csr, shard_range
from paper_1603_08390_b200.engine import ContractError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tweets():
    return synth.tweets(n=300_000, vocab=60_000, words=10, queries=96, k=100)


@pytest.fixture(scope="module")
def whole(tweets, gpu):
    ix = DeviceIndex.from_csr(tweets.csr, device=gpu)
    r = ix.query(tweets.queries)
    ix.close()
    return r


def same(a, b):
    assert np.array_equal(a.length, b.length) and np.array_equal(a.threshold, b.threshold)
    for q in range(a.length.shape[0]):
        assert a.row(q) == b.row(q), f"query {q}"
    assert hash_results(a.qid, a.threshold, a.length, a.ids, a.counts) == \
        hash_results(b.qid, b.threshold, b.length, b.ids, b.counts)


@pytest.mark.parametrize("shards", [1, 2, 3, 4, 8])
def test_group_equals_whole_index(tweets, whole, gpu, shards):
    g = DeviceGroup.from_csr(tweets.csr, [gpu] * shards, exchange=N.GENIE_EXCHANGE_PEER)
    assert g.num_shards == shards and g.exchange == N.GENIE_EXCHANGE_PEER
    r = g.query(tweets.queries, timings=True)
    same(r, whole)
    assert r.timings["total_ns"] >= r.timings["merge_ns"]
    assert r.stats["postings"] > 0
    g.close()


def test_group_equals_oracle(tweets, gpu):
    want = Oracle().index(tweets.csr).execute(tweets.queries)
    g = DeviceGroup.from_csr(tweets.csr, [gpu] * 3)
    same(g.query(tweets.queries), want)
    g.close()


def test_group_nccl_exchange_one_shard(tweets, whole, gpu):
    """ncclCommInitAll over the group's devices + ncclAllGather (1 rank here;
    the same calls serve 8 NVLink peers)."""
    g = DeviceGroup.from_csr(tweets.csr, [gpu], exchange=N.GENIE_EXCHANGE_NCCL)
    assert g.exchange == N.GENIE_EXCHANGE_NCCL
    same(g.query(tweets.queries), whole)
    g.close()


def test_nccl_needs_distinct_devices(tweets, gpu):
    with pytest.raises(ContractError, match="distinct device"):
        DeviceGroup.from_csr(tweets.csr, [gpu, gpu], exchange=N.GENIE_EXCHANGE_NCCL)


def test_group_from_partition_indexes(tweets, whole, gpu):
    """execute_partitioned's shape: independently built partitions (local ids)
    with their id offsets, borrowed by the group."""
    n, P = tweets.csr.n, 4
    parts, offs = [], []
    for p in range(P):
        lo, hi = shard_range(n, p, P)
        parts.append(DeviceIndex.from_csr(shard_csr(tweets.csr, lo, hi), device=gpu))
        offs.append(lo)
    g = DeviceGroup.from_indexes(parts, offs)
    same(g.query(tweets.queries), whole)
    g.close()
    # overlapping partitions report an object twice: merge_topk's ContractError
    dup = DeviceGroup.from_indexes([parts[0], parts[0]], [0, 0])
    with pytest.raises(ContractError, match="more than one partition"):
        dup.query(tweets.queries)
    dup.close()


def test_group_multi_tile_and_knobs(gpu):
    ds = synth.tweets(n=2_000_000, vocab=200_000, words=10, queries=64, k=100)
    want = DeviceIndex.from_csr(ds.csr, device=gpu).query(ds.queries)
    from paper_1603_08390_b200 import config
    g = DeviceGroup.from_csr(ds.csr, [gpu] * 2)
    for cfg in (config(), config(tile_bytes=32768), config(span_chunk=512)):
        same(g.query(ds.queries, cfg), want)
    g.close()
