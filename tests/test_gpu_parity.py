"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bit-exact: entries, thresholds and hash_results."""
import numpy as np
import pytest

from paper_1603_08390_b200 import DeviceIndex, config, synth

pytestmark = pytest.mark.gpu


def assert_same(got, want, label=""):
    assert np.array_equal(got.length, want.length), f"{label}: lengths differ"
    assert np.array_equal(got.threshold, want.threshold), f"{label}: thresholds differ"
    for q in range(len(got.length)):
        assert got.row(q) == want.row(q), f"{label}: query {q} differs"


@pytest.mark.parametrize("seed", range(12))
def test_random_instances_match_oracle(gpu, oracle, seed):
    ds = synth.random_instance(n=50 + 97 * seed, queries=16, seed=seed + 1)
    want = oracle.index(ds.csr).execute(ds.queries)
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    for sel in (0, 1):
        got = ix.query(ds.queries, config(selector=sel))
        assert_same(got, want, f"seed {seed} selector {sel}")


def test_adult_full_config(gpu, oracle):
    ds = synth.adult()
    want = oracle.index(ds.csr).execute(ds.queries)
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    got = ix.query(ds.queries, timings=True)
    assert_same(got, want, "adult")
    assert got.hash() == oracle.hash_results(want.qid, want.threshold, want.length, want.ids, want.counts)
    assert got.stats["postings"] == int(want.postings.sum())


@pytest.mark.parametrize("tile_bytes", [0, 8192, 65536])
def test_tweets_small_multi_tile(gpu, oracle, tile_bytes):
    ds = synth.tweets(n=300_000, vocab=100_000, words=10, queries=96, k=100)
    want = oracle.index(ds.csr).execute(ds.queries)
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    for sel in (0, 1):
        got = ix.query(ds.queries, config(selector=sel, tile_bytes=tile_bytes))
        assert_same(got, want, f"tweets tile {tile_bytes} sel {sel}")
