"""GPU parity: the CUDA path (through the C ABI) against the reference's own
results (golden fixtures) and the CPU oracle on the same seeded inputs.
Bit-exact: entries, thresholds and hash_results (engine.hpp:141-153)."""
import json
from pathlib import Path

import numpy as np
import pytest

from paper_1603_08390_b200 import CSR, ContractError, DeviceIndex, QueryBatch, config, merge_lists, synth
from tests.golden_util import config_dataset

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def assert_same(got, want, label=""):
    assert np.array_equal(got.length, want.length), f"{label}: lengths differ"
    assert np.array_equal(got.threshold, want.threshold), f"{label}: thresholds differ"
    for q in range(len(got.length)):
        assert got.row(q) == want.row(q), f"{label}: query {q} differs"


def test_golden_instances_equal_reference(gpu):
    g = np.load(GOLD / "random_instances.npz")
    for i in range(int(g["count"][0])):
        p = f"i{i}_"
        csr = CSR(int(g[p + "csr_n"][0]), g[p + "keys"], g[p + "key_off"], g[p + "postings"])
        qb = QueryBatch(*(g[p + "q_" + f] for f in ("qid", "k", "item_off", "dim", "lo", "hi")))
        ix = DeviceIndex.from_csr(csr, device=gpu)
        for sel in (0, 1, 2):
            r = ix.query(qb, config(selector=sel), stride=g[p + "ids"].shape[1])
            assert np.array_equal(r.length, g[p + "len"]) and np.array_equal(r.threshold, g[p + "thr"]), (i, sel)
            for q in range(len(qb)):
                n = int(r.length[q])
                assert np.array_equal(r.ids[q, :n], g[p + "ids"][q, :n]), (i, q, sel)
                assert np.array_equal(r.counts[q, :n], g[p + "counts"][q, :n]), (i, q, sel)
            assert r.hash() == int(g[p + "hash"][0])


@pytest.mark.parametrize("name", ["adult", "tweets_200k", "tweets_1m"])
def test_config_hash_equals_reference(gpu, name):
    want = json.loads((GOLD / "configs.json").read_text())[name]
    ds = config_dataset(name)
    got = DeviceIndex.from_csr(ds.csr, device=gpu).query(ds.queries)
    assert f"{got.hash():#018x}" == want["hash"]


@pytest.mark.parametrize("seed", range(10))
def test_random_instances_match_oracle(gpu, oracle, seed):
    ds = synth.random_instance(n=50 + 997 * seed, dims=4, tokens=8 + seed, max_kw=6, queries=24, max_items=5,
                               max_span=3, max_k=120, seed=seed + 1)
    want = oracle.index(ds.csr).execute(ds.queries)
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    for sel in (0, 1):
        assert_same(ix.query(ds.queries, config(selector=sel)), want, f"seed {seed} selector {sel}")


def test_adult_full_config(gpu, oracle):
    ds = synth.adult()
    want = oracle.index(ds.csr).execute(ds.queries)
    got = DeviceIndex.from_csr(ds.csr, device=gpu).query(ds.queries, timings=True, want_bound=True)
    assert_same(got, want, "adult")
    assert np.array_equal(got.bound, want.bound)
    assert got.stats["postings"] == int(want.postings.sum())
    t = got.timings
    assert t["lookup_ns"] + t["match_ns"] + t["select_ns"] + t["merge_ns"] <= t["total_ns"]


@pytest.mark.parametrize("tile_bytes", [0, 4096, 8192, 65536, 131072])
def test_tweets_multi_tile(gpu, oracle, tile_bytes):
    ds = synth.tweets(n=300_000, vocab=100_000, words=10, queries=96, k=100)
    want = oracle.index(ds.csr).execute(ds.queries)
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    for sel in (0, 1):
        assert_same(ix.query(ds.queries, config(selector=sel, tile_bytes=tile_bytes)), want,
                    f"tweets tile {tile_bytes} sel {sel}")


def test_scheduler_knobs_are_result_invariant(gpu):
    # test_engine.cpp:134-157: results independent of the decomposition knobs
    ds = synth.tweets(n=120_000, vocab=20_000, words=10, queries=40, k=64)
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    base = ix.query(ds.queries).hash()
    for chunk in (128, 1000, 4096, 65536):
        for tb in (16384, 65536):
            for cps in (0, 1):
                for sel in (0, 1, 2):
                    h = ix.query(ds.queries, config(selector=sel, span_chunk=chunk, tile_bytes=tb,
                                                    ctas_per_sm=cps)).hash()
                    assert h == base, (chunk, tb, cps, sel)
    with pytest.raises(ContractError, match="span_chunk and max_spans_per_task must be positive"):
        ix.query(ds.queries, config(span_chunk=0))


def test_wide_counters_w8_w16(gpu, oracle):
    # many items push max_count_bound past 15 (W=8) and 255 (W=16)
    ds = synth.random_instance(n=3000, dims=2, tokens=4, max_kw=8, queries=30, max_items=400, max_span=3,
                               max_k=50, seed=77)
    want = oracle.index(ds.csr).execute(ds.queries)
    assert want.bound.max() > 255 and (want.bound < 255).any()
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    for sel in (0, 1):
        for tb in (0, 4096):
            assert_same(ix.query(ds.queries, config(selector=sel, tile_bytes=tb)), want, f"wide {sel} {tb}")


@pytest.mark.parametrize("k,tile_bytes", [(1000, 4096), (20000, 0), (20000, 4096), (10**6, 0)])
def test_large_k_and_large_unions(gpu, oracle, k, tile_bytes):
    ds = synth.random_instance(n=50_000, dims=3, tokens=6, max_kw=5, queries=6, max_items=4, max_span=2, max_k=1,
                               seed=9)
    qb = ds.queries
    qb.k[:] = k
    want = oracle.index(ds.csr).execute(qb, stride=min(k, 60_000))
    got = DeviceIndex.from_csr(ds.csr, device=gpu).query(qb, config(tile_bytes=tile_bytes), stride=min(k, 60_000))
    assert_same(got, want, f"k={k}")


def test_edge_cases(gpu, oracle):
    # absent dims/tokens, duplicated and overlapping items, full-domain item, k > n, k = 1
    objs = [[(0, 1), (1, 2), (2, 1)], [(0, 2), (1, 1), (2, 2)], [(0, 1), (1, 2), (2, 2)], []]
    off = np.cumsum([0] + [len(o) for o in objs]).astype(np.uint64)
    csr = synth.csr_from_objects(4, off, np.array([d for o in objs for d, _ in o], np.uint16),
                                 np.array([t for o in objs for _, t in o], np.uint32))
    queries = [(0, 1, [(0, 1, 2), (1, 1, 1), (2, 2, 3)]),      # running example -> (1,3) thr 3
               (1, 10, [(9, 0, 100)]),                          # absent dim
               (2, 2, [(0, 1, 1), (0, 1, 1), (0, 0, 5)]),       # duplicate + overlapping items
               (3, 5, [(2, 0, 0xFFFFFFFF)]),                    # full domain, k > n
               (4, 4, [(1, 7, 9)]),                             # absent tokens, k == n
               (7, 3, [(0, 2, 2), (1, 1, 2), (2, 0, 1)])]
    off = np.cumsum([0] + [len(q[2]) for q in queries]).astype(np.uint64)
    its = [it for q in queries for it in q[2]]
    qb = QueryBatch([q[0] for q in queries], [q[1] for q in queries], off, [i[0] for i in its], [i[1] for i in its],
                    [i[2] for i in its])
    want = oracle.index(csr).execute(qb)
    got = DeviceIndex.from_csr(csr, device=gpu).query(qb)
    assert_same(got, want, "edges")
    assert got.row(0) == [(1, 3)] and got.threshold[0] == 3
    assert got.row(1) == [] and got.threshold[1] == 0
    assert got.row(2)[0] == (0, 3)
    assert got.threshold[3] == 0 and got.length[3] == 3
    assert list(got.qid) == [0, 1, 2, 3, 4, 7]


def test_empty_batch_and_empty_index(gpu):
    ds = synth.random_instance(n=100, seed=3)
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    empty = QueryBatch([], [], [0], [], [], [])
    r = ix.query(empty)
    assert r.length.shape == (0,)
    e = DeviceIndex.from_csr(CSR(0, np.zeros(0, np.uint64), np.zeros(1, np.uint64), np.zeros(0, np.uint32)),
                             device=gpu)
    r = e.query(ds.queries)
    assert np.all(r.length == 0) and np.all(r.threshold == 0)


def test_contract_errors(gpu):
    ds = synth.random_instance(n=100, seed=3)
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    bad = QueryBatch([5], [0], [0, 1], [0], [0], [0])
    with pytest.raises(ContractError, match="Query 5: k must be >= 1"):
        ix.query(bad)
    with pytest.raises(ContractError, match="Query 6: no items"):
        ix.query(QueryBatch([6], [1], [0, 0], [], [], []))
    with pytest.raises(ContractError, match="lo 3 > hi 2"):
        ix.query(QueryBatch([6], [1], [0, 1], [0], [3], [2]))
    # a bound above 0xffff is a ContractError at setup (engine.hpp:230-233)
    d, t = int(ds.csr.keys[0]) >> 32, int(ds.csr.keys[0]) & 0xFFFFFFFF
    n_items = 70_000
    big = QueryBatch([0, 41], [1, 1], [0, 1, 1 + n_items], [d] * (1 + n_items), [t] * (1 + n_items),
                     [t] * (1 + n_items))
    with pytest.raises(ContractError, match=r"query 41 \(setup\): match-count bound 70000 exceeds the counter range"):
        ix.query(big)


def test_shards_merge_equals_whole(gpu, oracle):
    # execute_partitioned semantics (engine.hpp:308-347) with device shards + device merge
    ds = synth.tweets(n=200_000, vocab=30_000, words=10, queries=50, k=100)
    want = oracle.index(ds.csr).execute(ds.queries)
    world = 3
    Q, K = len(ds.queries), 100
    ids = np.zeros((Q, world, K), np.uint32)
    cnt = np.zeros((Q, world, K), np.uint32)
    lens = np.zeros((Q, world), np.uint32)
    from paper_1603_08390_b200.dist import shard_range
    for r in range(world):
        lo, hi = shard_range(ds.csr.n, r, world)
        sh = DeviceIndex.shard(ds.csr, lo, hi, device=gpu)
        assert sh.id_offset == lo and sh.num_objects == hi - lo
        res = sh.query(ds.queries)
        ids[:, r], cnt[:, r], lens[:, r] = res.ids, res.counts, res.length
    oi, oc, ol, ot = merge_lists(ids, cnt, lens, ds.queries.k, device=gpu)
    assert np.array_equal(ol, want.length) and np.array_equal(ot, want.threshold)
    for q in range(Q):
        n = int(ol[q])
        assert np.array_equal(oi[q, :n], want.ids[q, :n]) and np.array_equal(oc[q, :n], want.counts[q, :n])
    # duplicate ids across lists -> ContractError
    ids[0, 1, 0] = ids[0, 0, 0]
    cnt[0, 1, 0] = 1
    lens[0, 1] = max(lens[0, 1], 1)
    with pytest.raises(ContractError):
        merge_lists(ids, cnt, lens, ds.queries.k, device=gpu)


def test_device_api_equals_host_api(gpu):
    import torch

    ds = synth.tweets(n=150_000, vocab=20_000, words=10, queries=64, k=100)
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    host = ix.query(ds.queries)
    qb, dev = ds.queries, torch.device("cuda", gpu)
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        d = {"qid": torch.from_numpy(qb.qid.astype(np.int32)).to(dev), "k": torch.from_numpy(qb.k.astype(np.int32)).to(dev),
             "item_off": torch.from_numpy(qb.item_off.astype(np.int64)).to(dev),
             "dim": torch.from_numpy(qb.dim.astype(np.int16)).to(dev), "lo": torch.from_numpy(qb.lo.astype(np.int32)).to(dev),
             "hi": torch.from_numpy(qb.hi.astype(np.int32)).to(dev),
             "out": torch.zeros((len(qb), 100, 2), dtype=torch.int32, device=dev),
             "out_len": torch.zeros(len(qb), dtype=torch.int32, device=dev),
             "out_thr": torch.zeros(len(qb), dtype=torch.int32, device=dev),
             "max_k": 100, "total_items": qb.num_items, "stride": 100}
        for _ in range(4):
            ix.query_device(d, stream=s.cuda_stream)
            if not ix.status().get("retry"):
                break
    s.synchronize()
    out = d["out"].cpu().numpy().view(np.uint32)
    assert np.array_equal(d["out_len"].cpu().numpy(), host.length.astype(np.int32))
    assert np.array_equal(d["out_thr"].cpu().numpy(), host.threshold.astype(np.int32))
    for q in range(len(qb)):
        n = int(host.length[q])
        assert np.array_equal(out[q, :n, 0], host.ids[q, :n]) and np.array_equal(out[q, :n, 1], host.counts[q, :n])


def test_device_dim_stats_match_oracle(gpu, oracle):
    ds = synth.random_instance(n=5000, dims=6, tokens=9, max_kw=8, queries=1, seed=12)
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    dm = ix.dim_stats()
    oi = oracle.index(ds.csr)
    for d in range(8):
        assert dm[d] == oi.max_multiplicity(d)
    back = ix.export()
    assert np.array_equal(back.keys, ds.csr.keys) and np.array_equal(back.postings, ds.csr.postings)


@pytest.mark.parametrize("density", ["0", "0.002", "0.05", "0.125", "0.5"])
def test_dense_containers_are_result_invariant(gpu, oracle, density, monkeypatch):
    # lists above the density threshold carry a bitmap container that replaces
    # their posting scan; any threshold must give the oracle's results
    monkeypatch.setenv("GENIE_DENSE_MIN_DENSITY", density)
    for ds in (synth.tweets(n=250_000, vocab=20_000, words=10, queries=64, k=100),
               synth.random_instance(n=40_000, dims=3, tokens=5, max_kw=8, queries=40, max_items=40, max_span=2,
                                     max_k=60, seed=5)):
        want = oracle.index(ds.csr).execute(ds.queries)
        ix = DeviceIndex.from_csr(ds.csr, device=gpu)
        for sel in (0, 1):
            for tb in (0, 4096, 32768):
                assert_same(ix.query(ds.queries, config(selector=sel, tile_bytes=tb)), want,
                            f"density {density} sel {sel} tile {tb}")


@pytest.mark.parametrize("seed", range(6))
def test_tie_heavy_many_tiles(gpu, oracle, seed, monkeypatch):
    # Few tokens per dim: long lists, and thousands of objects tied at the
    # k-th count.  Small tiles give each query dozens of (query, tile) items,
    # so later tiles start their gate above the lower tiles' counts (ties lose
    # on id) and the merge prunes below the published floor; every variant
    # must still equal the oracle bit for bit.
    ds = synth.random_instance(n=20_000 + 3001 * seed, dims=3, tokens=3 + seed % 3, max_kw=6, queries=32,
                               max_items=6, max_span=2, max_k=300, seed=100 + seed)
    want = oracle.index(ds.csr).execute(ds.queries)
    for density in ("0", "0.05"):
        monkeypatch.setenv("GENIE_DENSE_MIN_DENSITY", density)
        ix = DeviceIndex.from_csr(ds.csr, device=gpu)
        for tb in (4096, 8192, 0):
            for rep in range(2):  # concurrent tiles finish in a different order each run
                assert_same(ix.query(ds.queries, config(tile_bytes=tb)), want,
                            f"seed {seed} density {density} tile {tb} rep {rep}")


@pytest.mark.parametrize("tile_bytes", [4096, 16384, 0])
def test_many_spans_per_query(gpu, oracle, tile_bytes):
    # Range items over a dim of 1500 tokens: a query resolves to up to ~1200
    # keyword lists, more than one staging batch (256 spans), so the further
    # batches are staged block-wide; short lists also select the compact
    # (one id per lane) scan.  Multi-tile at the small tile sizes.
    rng = np.random.default_rng(77)
    n, ntok = 30_000, 1500
    kw = rng.integers(1, 4, size=n)
    off = np.concatenate([[0], np.cumsum(kw)]).astype(np.uint64)
    dims = rng.integers(0, 2, size=int(off[-1])).astype(np.uint16)
    toks = rng.integers(0, ntok, size=int(off[-1])).astype(np.uint32)
    # one keyword per (object, dim): drop duplicates by making dim 1 tokens distinct per object
    for i in range(n):
        a, b = int(off[i]), int(off[i + 1])
        dims[a:b] = np.arange(b - a) % 2
        if b - a == 3:
            dims[b - 1] = 2
    csr = synth.csr_from_objects(n, off, dims, toks)
    Q = 12
    qdim, qlo, qhi, qoff = [], [], [], [0]
    for q in range(Q):
        for _ in range(1 + q % 3):
            lo = int(rng.integers(0, ntok // 2))
            qdim.append(int(rng.integers(0, 2)))
            qlo.append(lo)
            qhi.append(min(ntok - 1, lo + int(rng.integers(200, 700))))
        qoff.append(len(qdim))
    qb = QueryBatch(np.arange(Q, dtype=np.uint32), np.array([1 + 37 * q for q in range(Q)], np.uint32),
                    np.array(qoff, np.uint64), np.array(qdim, np.uint16), np.array(qlo, np.uint32),
                    np.array(qhi, np.uint32))
    want = oracle.index(csr).execute(qb)
    ix = DeviceIndex.from_csr(csr, device=gpu)
    for sel in (0, 1):
        assert_same(ix.query(qb, config(selector=sel, tile_bytes=tile_bytes)), want, f"spans tile {tile_bytes} sel {sel}")


@pytest.mark.parametrize("tile_bytes", [4096, 16384])
def test_many_queries_grouped_cuts(gpu, oracle, tile_bytes):
    # ~72K (query, keyword list) spans in one batch: more spans than k_cut has
    # warps, so each warp resolves a group of spans lane-parallel and cuts
    # their flattened (span, tile boundary) pairs (the C4 shape: many short
    # single-token items per query, many tiles per query).
    rng = np.random.default_rng(5)
    n, ndim, ntok, Q, m = 200_000, 32, 128, 3000, 24
    off = (np.arange(n + 1, dtype=np.uint64) * ndim)
    dims = np.tile(np.arange(ndim, dtype=np.uint16), n)
    toks = rng.integers(0, ntok, size=n * ndim).astype(np.uint32)
    csr = synth.csr_from_objects(n, off, dims, toks)
    qdim = np.concatenate([rng.permutation(ndim)[:m] for _ in range(Q)]).astype(np.uint16)
    qtok = rng.integers(0, ntok, size=Q * m).astype(np.uint32)
    qb = QueryBatch(np.arange(Q, dtype=np.uint32), rng.integers(1, 150, size=Q).astype(np.uint32),
                    (np.arange(Q + 1, dtype=np.uint64) * m), qdim, qtok, qtok)
    want = oracle.index(csr).execute(qb)
    ix = DeviceIndex.from_csr(csr, device=gpu)
    assert_same(ix.query(qb, config(tile_bytes=tile_bytes)), want, f"grouped cuts tile {tile_bytes}")


def test_mcix_image_loads_into_the_device_index(gpu, oracle, tmp_path):
    # load_index (index_io.hpp:148-154) straight into device memory: the same
    # CSR back, the same answers as the oracle
    from paper_1603_08390_b200 import engine as E
    from paper_1603_08390_b200 import mcx

    ds = synth.tweets(n=120_000, vocab=30_000, words=10, queries=48, k=100)
    img = E.mcix_serialize(ds.csr, 4096)
    ix = DeviceIndex.from_mcix(img, device=gpu)
    back = ix.export()
    assert np.array_equal(back.keys, ds.csr.keys) and np.array_equal(back.postings, ds.csr.postings)
    want = oracle.index(ds.csr).execute(ds.queries)
    assert_same(ix.query(ds.queries), want, "mcix")
    path = tmp_path / "tweets.mcix"
    mcx.save_index(mcx.InvertedIndex(ds.csr, 4096), str(path))
    loaded = mcx.load_index(str(path))
    assert np.array_equal(loaded.csr.key_off, ds.csr.key_off)
    assert_same(DeviceIndex.from_mcix(str(path), device=gpu).query(ds.queries), want, "mcix file")


@pytest.mark.parametrize("seed", range(3))
def test_device_build_equals_host_build(gpu, oracle, seed):
    # build_index (index.hpp:190-250) on the device: the same CSR as the host
    # build, the same answers
    rng = np.random.default_rng(seed)
    n = 20_000 + 7_000 * seed
    kw = rng.integers(0, 12, size=n)
    off = np.concatenate([[0], np.cumsum(kw)]).astype(np.uint64)
    dims = np.empty(int(off[-1]), np.uint16)
    toks = np.empty(int(off[-1]), np.uint32)
    for o in range(n):  # distinct (dim, token) per object
        a, b = int(off[o]), int(off[o + 1])
        code = rng.choice(4 * 300, size=b - a, replace=False)
        dims[a:b] = code // 300
        toks[a:b] = code % 300 + (seed * 1000)
    host = synth.csr_from_objects(n, off, dims, toks)
    ix = DeviceIndex.build(n, off, dims, toks, device=gpu)
    back = ix.export()
    assert np.array_equal(back.keys, host.keys) and np.array_equal(back.key_off, host.key_off)
    assert np.array_equal(back.postings, host.postings)
    ds = synth.random_instance(n=10, seed=1)  # only for a query shape
    qb = QueryBatch(np.arange(8, dtype=np.uint32), np.full(8, 50, np.uint32), np.arange(9, dtype=np.uint64) * 2,
                    np.array([0, 1] * 8, np.uint16), np.array([seed * 1000 + 5 * i for i in range(16)], np.uint32),
                    np.array([seed * 1000 + 5 * i + 40 for i in range(16)], np.uint32))
    assert_same(ix.query(qb), oracle.index(host).execute(qb), f"device build {seed}")
    dup_dims, dup_toks = dims.copy(), toks.copy()
    j = int(np.argmax(kw >= 2))
    a = int(off[j])
    dup_dims[a + 1], dup_toks[a + 1] = dup_dims[a], dup_toks[a]
    with pytest.raises(ContractError, match="duplicate keyword"):
        DeviceIndex.build(n, off, dup_dims, dup_toks, device=gpu)


def test_cuda_graph_replay_equals_direct_launches(gpu):
    """GENIE_FLAG_GRAPH: the batch pipeline captured once and replayed while
    nothing it depends on changes; new buffers / a grown workspace re-capture.
    Every replay's results equal the host API's."""
    import torch

    from paper_1603_08390_b200 import config

    dev = torch.device("cuda", gpu)
    s = torch.cuda.Stream(dev)

    def dev_batch(qb):
        with torch.cuda.stream(s):
            return {"qid": torch.from_numpy(qb.qid.astype(np.int32)).to(dev),
                    "k": torch.from_numpy(qb.k.astype(np.int32)).to(dev),
                    "item_off": torch.from_numpy(qb.item_off.astype(np.int64)).to(dev),
                    "dim": torch.from_numpy(qb.dim.astype(np.int16)).to(dev),
                    "lo": torch.from_numpy(qb.lo.astype(np.int32)).to(dev),
                    "hi": torch.from_numpy(qb.hi.astype(np.int32)).to(dev),
                    "out": torch.zeros((len(qb), 100, 2), dtype=torch.int32, device=dev),
                    "out_len": torch.zeros(len(qb), dtype=torch.int32, device=dev),
                    "out_thr": torch.zeros(len(qb), dtype=torch.int32, device=dev),
                    "max_k": 100, "total_items": qb.num_items, "stride": 100}

    def check(d, host):
        s.synchronize()
        out = d["out"].cpu().numpy().view(np.uint32)
        assert np.array_equal(d["out_len"].cpu().numpy(), host.length.astype(np.int32))
        assert np.array_equal(d["out_thr"].cpu().numpy(), host.threshold.astype(np.int32))
        for q in range(host.length.shape[0]):
            n = int(host.length[q])
            assert np.array_equal(out[q, :n, 0], host.ids[q, :n]) and np.array_equal(out[q, :n, 1], host.counts[q, :n])

    ds = synth.tweets(n=400_000, vocab=40_000, words=10, queries=128, k=100)
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    host = ix.query(ds.queries)
    cfg = config(graph=True, stage_events=True)  # stage events replay as external event nodes
    d = dev_batch(ds.queries)
    for _ in range(4):  # first call may grow the workspace (retry), then the graph settles
        ix.query_device(d, cfg, stream=s.cuda_stream)
        if not ix.status().get("retry"):
            break
    settled = ix.graph_captures()
    for _ in range(5):
        d["out"].zero_()
        ix.query_device(d, cfg, stream=s.cuda_stream)
        assert not ix.status().get("retry")
        check(d, host)
    assert ix.graph_captures() == settled  # pure replays
    st = ix.stage_ns()
    assert st["match_ns"] > 0 and st["lookup_ns"] > 0
    # a different batch (new buffers): re-captured, still exact
    ds2 = synth.tweets(n=400_000, vocab=40_000, words=10, queries=96, k=100, seed=99)
    host2 = DeviceIndex.from_csr(ds.csr, device=gpu).query(ds2.queries)
    d2 = dev_batch(ds2.queries)
    for _ in range(4):
        ix.query_device(d2, cfg, stream=s.cuda_stream)
        if not ix.status().get("retry"):
            break
    check(d2, host2)
    assert ix.graph_captures() > settled


@pytest.mark.parametrize("tile_bytes", [0, 16384])
def test_key_cut_table_equals_searches(gpu, oracle, tile_bytes):
    """The first batch of a width class cuts lists by binary search; later
    batches read the per-key cut table built from it (k_keycut).  Both, and a
    tile-size change (table rebuilt), give the oracle's answer."""
    from paper_1603_08390_b200 import config

    ds = synth.tweets(n=600_000, vocab=50_000, words=10, queries=96, k=100)
    want = oracle.index(ds.csr).execute(ds.queries)
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    for cfg in (config(tile_bytes=tile_bytes), config(tile_bytes=tile_bytes), config(tile_bytes=8192),
                config(tile_bytes=tile_bytes)):
        got = ix.query(ds.queries, cfg)
        assert np.array_equal(got.length, want.length) and np.array_equal(got.threshold, want.threshold)
        for q in range(len(ds.queries)):
            assert got.row(q) == want.row(q)
    ix.close()


def test_host_api_graph_with_pinned_buffers(gpu):
    """genie_query_batch with GENIE_FLAG_GRAPH and page-locked buffers: uploads,
    pipeline and read-backs replay as one graph; results equal the direct call;
    pageable buffers take the direct path."""
    import torch

    from paper_1603_08390_b200 import config
    from paper_1603_08390_b200.engine import QueryBatch

    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    ds = synth.tweets(n=400_000, vocab=40_000, words=10, queries=128, k=100)
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    want = ix.query(ds.queries)
    qb = ds.queries
    hb = QueryBatch(pin(qb.qid), pin(qb.k), pin(qb.item_off), pin(qb.dim), pin(qb.lo), pin(qb.hi))
    out = (pin(np.zeros((len(qb), 100, 2), np.uint32)), pin(np.zeros(len(qb), np.uint32)),
           pin(np.zeros(len(qb), np.uint32)))
    cfg = config(graph=True)
    before = ix.graph_captures()
    for i in range(4):
        out[0][:] = 0
        got = ix.query(hb, cfg, stride=100, out=out, timings=(i == 3))
        assert np.array_equal(got.length, want.length) and np.array_equal(got.threshold, want.threshold)
        for q in range(len(qb)):
            assert got.row(q) == want.row(q)
        assert got.stats["counter_bytes"] == want.stats["counter_bytes"]
    assert got.timings["match_ns"] > 0
    assert ix.graph_captures() - before <= 3  # first use, (timed variant), not every call
    pageable = ix.query(qb, cfg)  # not pinned: direct launches, same answer
    assert pageable.hash() == want.hash()
